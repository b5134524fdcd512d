#!/bin/bash
python tools/pulls.py 2 8 1e7 40
python tools/pulls.py 4 8 1e8 20
python tools/pulls.py 5 8 1e7 40
python tools/pulls.py 6 8 1e7 40

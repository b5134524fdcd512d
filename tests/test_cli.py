"""The benchmark CLI (paper_2202_01753_b200.bench_cli), ported from the
reference's tests/test_cli.cpp.  summarize and the usage errors are host-only
(CPU); run/sweep need the GPU."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

HEADER = ("integrand,dims,tau_rel,run,seed,estimate,sigma,chi2_dof,converged,"
          "true_value,rel_error,iterations,total_samples,wall_ms")
BENCH = [sys.executable, "-m", "paper_2202_01753_b200.bench_cli"]


def run(args, **kw):
    return subprocess.run(BENCH + args, capture_output=True, text=True, cwd=ROOT, timeout=600, **kw)


def strip_wall(text):
    return "\n".join(",".join(ln.split(",")[:13]) for ln in text.splitlines())


def test_usage_errors_exit_1_and_help_0():
    # test_cli.cpp:104-114 (the integrand/dims checks fail before any GPU work)
    assert run(["run", "--integrand", "f9", "--dim", "2"]).returncode == 1
    assert run(["run"]).returncode == 1
    assert run(["run", "--integrand", "f4", "--dim", "2", "--variant", "bogus"]).returncode == 1
    assert run([]).returncode == 1
    assert run(["summarize", "/nonexistent_input.csv"]).returncode == 1
    assert run(["run", "--integrand", "fA", "--dim", "3"]).returncode == 1
    assert run(["--help"]).returncode == 0
    assert run(["run", "--help"]).returncode == 0


def test_summarize_quartiles(tmp_path):
    # test_cli.cpp:169-217
    p = tmp_path / "in.csv"
    p.write_text(HEADER + "\n" +
                 "f4,2,0.001,0,1,1.0,0.01,0.5,1,1.0,0.1,5,1000,1.5\n"
                 "f4,2,0.001,1,2,1.0,0.01,0.5,1,1.0,0.3,5,1000,1.5\n"
                 "f4,2,0.001,2,3,1.0,0.01,0.5,1,1.0,0.2,5,1000,1.5\n"
                 "f4,2,0.001,3,4,1.0,0.01,0.5,1,1.0,0.4,5,1000,1.5\n"
                 "f4,2,0.001,4,5,1.0,0.01,9.9,0,1.0,0.9,5,1000,1.5\n"
                 "fB,9,0.001,0,1,1.0,0.01,0.5,1,,,5,1000,1.5\n")
    r = run(["summarize", str(p)])
    assert r.returncode == 0
    lines = r.stdout.splitlines()
    assert len(lines) == 3
    assert lines[0] == ("integrand,dims,tau_rel,runs,converged,convergence_rate,"
                        "min_rel_error,q1_rel_error,median_rel_error,q3_rel_error,max_rel_error")
    g1 = lines[1].split(",")
    assert g1[:2] == ["f4", "2"] and g1[3] == "5" and g1[4] == "4" and abs(float(g1[5]) - 0.8) < 1e-12
    for got, want in zip(g1[6:], [0.1, 0.175, 0.25, 0.325, 0.4]):
        assert abs(float(got) - want) < 1e-12 * want
    g2 = lines[2].split(",")
    assert g2[0] == "fB" and g2[4] == "1" and all(x == "" for x in g2[6:]) and len(g2) == 11
    out = tmp_path / "out.csv"
    assert run(["summarize", str(p), "--out", str(out)]).returncode == 0
    assert out.read_text() == r.stdout


def test_summarize_rejects_bad_inputs(tmp_path):
    # test_cli.cpp:219-235
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b,c\n")
    assert run(["summarize", str(bad)]).returncode == 1
    bad.write_text(HEADER + "\nf4,2,0.001,0,1,1.0\n")
    assert run(["summarize", str(bad)]).returncode == 1


@pytest.mark.gpu
def test_run_row_and_exit_codes():
    # test_cli.cpp:66-102
    r = run(["run", "--integrand", "f4", "--dim", "2", "--maxcalls", "4000", "--tau-rel", "0.5", "--seed", "3"])
    assert r.returncode == 0
    lines = r.stdout.splitlines()
    assert lines[0] == HEADER and len(lines) == 2
    f = lines[1].split(",")
    assert len(f) == 14 and f[0] == "f4" and f[1] == "2" and f[3] == "0" and f[4] == "3" and f[8] == "1"
    assert float(f[6]) > 0 and float(f[10]) >= 0 and int(f[12]) % 3872 == 0
    r = run(["run", "--integrand", "f4", "--dim", "2", "--maxcalls", "2000", "--tau-rel", "1e-9", "--itmax", "3",
             "--ita", "2"])
    assert r.returncode == 2
    f = r.stdout.splitlines()[1].split(",")
    assert f[8] == "0" and f[11] == "3"


@pytest.mark.gpu
def test_repeatable_and_out_file(tmp_path):
    # test_cli.cpp:116-131
    cmd = ["run", "--integrand", "f5", "--dim", "3", "--maxcalls", "3000", "--seed", "11", "--tau-rel", "1e-2"]
    a = run(cmd)
    b = run(cmd + ["--workers", "3"])
    assert a.returncode == b.returncode and strip_wall(a.stdout) == strip_wall(b.stdout)
    out = tmp_path / "o.csv"
    c = run(cmd + ["--out", str(out)])
    assert c.returncode == a.returncode and c.stdout == ""
    assert strip_wall(out.read_text()) == strip_wall(a.stdout)


@pytest.mark.gpu
def test_sweep_schedule(tmp_path):
    # test_cli.cpp:133-167
    out = tmp_path / "s.csv"
    r = run(["sweep", "--integrand", "f4", "--dim", "1", "--maxcalls", "1000", "--runs", "4", "--seed", "7", "--out",
             str(out)])
    assert r.returncode == 0
    lines = out.read_text().splitlines()
    assert lines[0] == HEADER and (len(lines) - 1) % 4 == 0
    levels = (len(lines) - 1) // 4
    assert 1 <= levels <= 9
    tau = 1e-3
    for level in range(levels):
        conv = 0
        for i in range(4):
            f = lines[1 + level * 4 + i].split(",")
            assert len(f) == 14 and abs(float(f[2]) - tau) <= 1e-12 * tau and f[3] == str(i)
            assert int(f[4]) == 7 + level * 4 + i
            conv += f[8] == "1"
        if level + 1 < levels:
            assert conv * 2 >= 4
        else:
            assert conv * 2 < 4 or levels == 9
        tau /= 5.0


@pytest.mark.gpu
def test_scale_subcommand(tmp_path):
    """bench.py --scale: the CLI's scale sweep with the reference CPU column
    filled in the same run (the library never runs a CPU path itself)."""
    out = tmp_path / "scale.csv"
    r = subprocess.run([sys.executable, "bench.py", "--scale", str(out), "--scale-dims", "3,8",
                        "--scale-ncalls", "1e6,1e8"], capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    head = lines[0].split(",")
    assert len(lines) == 5 and lines[0].startswith("integrand,dims,maxcalls")
    col = {k: i for i, k in enumerate(head)}
    for ln in lines[1:]:
        f = ln.split(",")
        assert int(f[col["gpus"]]) == 1
        assert float(f[col["evals_per_s"]]) > 1e8
        # the reference CPU iteration on the host cores, in the same run
        assert int(f[col["cpu_threads"]]) >= 1 and float(f[col["cpu_evals_per_s"]]) > 0
        assert float(f[col["speedup"]]) > 1


@pytest.mark.gpu
def test_scale_subcommand_multi_rank(tmp_path):
    """The scale sweep under torchrun (world 2 sharing cuda:0 over gloo):
    the gpus column and the same cells."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "scale2.csv"
    env = dict(os.environ, MCB_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "-m",
                        "paper_2202_01753_b200.bench_cli", "scale", "--integrand", "f4", "--dims", "4",
                        "--ncalls", "1e7", "--out", str(out)],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = out.read_text().splitlines()
    assert len(lines) == 2
    f = dict(zip(lines[0].split(","), lines[1].split(",")))
    assert f["gpus"] == "2" and float(f["evals_per_s"]) > 1e8

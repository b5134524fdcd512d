VARS="base rz rzp rp" bash tools/gpu_k1var.sh > /dev/null
cat gpurun_out/k1var.txt | awk '{print $2, $3, $NF, $(NF-1)}'
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel --launch-skip 4 -c 1 -o /tmp/k1base tools/bin/k1bench_base 1000000000 1 1 0 4 > gpurun_out/ncu_k1base.log 2>&1
ncu -i /tmp/k1base.ncu-rep --page raw --csv > gpurun_out/k1base_raw.csv 2>/dev/null
ncu -i /tmp/k1base.ncu-rep --page details --csv > gpurun_out/k1base_details.csv 2>/dev/null
gzip -f gpurun_out/k1base_raw.csv
ls -la gpurun_out

mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:redrec_kernel -s 1 -c 1 -o gpurun_out/rr256_full -f python tools/perf_probe.py r256_redrec_b2048 > gpurun_out/ncu_rr.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/rr256_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/rr256_src.csv 2>/dev/null; echo src rc=$?

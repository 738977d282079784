# ncu --set full of the bird kernel at the 256^2 batch, source-correlated
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bird_kernel -s 1 -c 1 -o gpurun_out/bird_full -f python tools/perf_probe.py c4_bird_2048 > gpurun_out/ncu_b.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/bird_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/bird_src.csv 2>/dev/null

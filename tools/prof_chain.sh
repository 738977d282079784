# ncu --set full of the chain band kernel (C2, 1M chains), source-correlated
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_band -s 1 -c 1 -o gpurun_out/chain_full -f python tools/perf_probe.py c2_chains_1m > gpurun_out/ncu_c.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/chain_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/chain_src.csv 2>/dev/null; python tools/perf_probe.py c2_chains_1m | cut -c1-120

# ncu --set full of the red-rec executor at the bench batch (one launch), source-correlated
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:redrec_kernel -s 1 -c 1 -o gpurun_out/redrec_full -f python tools/perf_probe.py c4_redrec_2048 > gpurun_out/ncu_f1.log 2>&1; echo ncu rc=$?

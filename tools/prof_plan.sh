set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:redrec_plan_kernel -s 1 -c 1 -o gpurun_out/plan1 -f python tools/perf_probe.py c4_redrec_h153_1 > gpurun_out/ncu_p.log 2>&1; echo ncu rc=$?

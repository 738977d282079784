# ncu --set full of the batching kernel on C5 (bird 512^2 + batching, 4 instances)
set -x
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:batch_pipeline -s 0 -c 1 -o gpurun_out/batch_full -f python tools/perf_probe.py ${CASE:-c5_pipeline_4} > gpurun_out/ncu_bt.log 2>&1; echo ncu rc=$?

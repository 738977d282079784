# launch list + full capture of the batching kernel on C3 (bird 64^2 + batching, 4096 instances)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/perf_probe.py c3_pipeline_none > gpurun_out/ncu_c3l.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_pipeline -s 1 -c 1 -o gpurun_out/c3_batch_full -f python tools/perf_probe.py c3_pipeline_none > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/c3_batch_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c3_batch_src.csv 2>/dev/null

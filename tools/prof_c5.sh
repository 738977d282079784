# launch list + full capture of the batching kernel on C5 (bird 512^2 + batching, 4 instances)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/perf_probe.py c5_pipeline_4 > gpurun_out/ncu_c5l.log 2>&1; echo rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:batch_pipeline -s 1 -c 1 -o gpurun_out/c5_batch_full -f python tools/perf_probe.py c5_pipeline_4 > gpurun_out/ncu_c5.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/c5_batch_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c5_batch_src.csv 2>/dev/null

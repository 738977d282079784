# batching pipeline timings: move log forced on / off / auto
for m in 1 0; do echo "LOG=$m"; RECON_BATCH_LOG=$m python tools/perf_probe.py c3_pipeline_none c3_pipeline_coldir | cut -c1-90; done
echo auto; python tools/perf_probe.py c3_pipeline_none c3_pipeline_coldir c4_pipeline_redrec_64 c5_pipeline_4 | cut -c1-90
python -m pytest tests -m gpu -q -x 2>&1 | tail -1

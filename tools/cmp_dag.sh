# pipeline with the per-instance shared-memory DAG builder on / off
for m in 1 0; do echo "SMALL_DAG=$m"; RECON_SMALL_DAG=$m python tools/perf_probe.py c3_pipeline_none c3_pipeline_coldir | cut -c1-90; done
python -m pytest tests -m gpu -q -x 2>&1 | tail -2

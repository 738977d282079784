python -m pytest tests/test_batching_gpu.py -q -x 2>&1 | tail -1
timeout 600 python tools/perf_probe.py c5_pipeline_512 | cut -c1-110
timeout 600 python tools/perf_probe.py c5_pipeline_4 | cut -c1-110

# Round-end measurement refresh (one GPU): GPU tests, bench line, the bench's
# ncu launch list, and --set full captures of the top kernels.  Then run
# `python tools/prof_collect.py r01` here to write profiles/.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -1 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_l.log 2>&1; echo ncu-launches rc=$?
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:redrec_kernel -s 3 -c 1 -o gpurun_out/redrec_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_f1.log 2>&1; echo ncu-redrec rc=$?
timeout 900 ncu $F -k regex:redrec_plan_kernel -s 3 -c 1 -o gpurun_out/plan_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_f2.log 2>&1; echo ncu-plan rc=$?
timeout 900 ncu $F -k regex:bird_kernel -s 1 -c 1 -o gpurun_out/bird_full -f python tools/perf_probe.py c4_bird_2048 > gpurun_out/ncu_b.log 2>&1; echo ncu-bird rc=$?
timeout 900 ncu $F -k regex:chain_band -s 1 -c 1 -o gpurun_out/chain_full -f python tools/perf_probe.py c2_chains_1m > gpurun_out/ncu_c.log 2>&1; echo ncu-chain rc=$?
timeout 900 ncu $F -k regex:batch_pipeline -s 1 -c 1 -o gpurun_out/c3_batch_full -f python tools/perf_probe.py c3_pipeline_none > gpurun_out/ncu_c3.log 2>&1; echo ncu-batch rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/perf_probe.py c3_pipeline_none > gpurun_out/ncu_c3l.log 2>&1; echo ncu-c3-launches rc=$?
python tools/perf_probe.py c1_redrec c1_redrec_1 c2_chains_1m c3_bird_solve c3_pipeline_none c3_pipeline_coldir c4_redrec_h128_1 c4_redrec_h153_1 c4_bird_h153_1 c4_redrec_2048 c4_bird_2048 c4_pipeline_redrec_64 c5_bird_solve_1 c5_bird_solve_64 c5_pipeline_4 c4_json c5_json > gpurun_out/probe_all.jsonl 2> gpurun_out/probe_all.err; echo probe rc=$?

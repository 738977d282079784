set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -2 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_l.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:redrec_kernel -s 3 -c 1 -o gpurun_out/redrec_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_f1.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:redrec_plan_kernel -s 3 -c 1 -o gpurun_out/plan_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_f2.log 2>&1; echo ncu3 rc=$?

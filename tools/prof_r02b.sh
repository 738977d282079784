#!/bin/bash
# Round-2 final profiles (window phase, reduced DAG, early leap finishes), one
# B200 under gpurun; text summaries in gpurun_out/prof_r02b, copied to profiles/:
#  1. the full bench line
#  2. the bench's ncu launch list (gpu__time_duration, clocks not locked)
#  3. ncu --set full of the C5 pipeline kernels at 64 instances
#  4. the clock64 phase counters of the batching kernels (-DRECON_BATCH_PROF)
#  5. the checked build (tools/checked_run.sh)
cd "$(dirname "$0")/.."
O=gpurun_out/prof_r02b
mkdir -p $O
timeout 1500 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
grep '^{' $O/bench.log | tail -1 > $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-extras --no-cpu > $O/bench_under_ncu.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench_summary.txt 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on \
    -k regex:"batch_window|batch_pipeline_kernel|pl_walk|pl_mark2|bird_kernel|pl_compact" -c 6 \
    -o $O/c5_full -f python tools/perf_probe.py c5_pipeline_64 > $O/ncu_c5.log 2>&1; echo "c5 full rc=$?"
python tools/ncu_raw.py $O/c5_full.ncu-rep > $O/c5_full_raw.txt 2>&1
for k in batch_window batch_pipeline_kernel pl_walk pl_mark2 bird_kernel; do
    ncu -i $O/c5_full.ncu-rep --page source --csv --print-source cuda,sass -k regex:"$k" > $O/src.csv 2>/dev/null
    python tools/ncu_lines.py $O/src.csv 30 > $O/c5_lines_$k.txt 2>&1
done
rm -f $O/src.csv $O/*.ncu-rep
RECON_BUILD_TAG=prof RECON_NVCC_EXTRA=-DRECON_BATCH_PROF python paper_2504_06182_b200/build_native.py > $O/prof_build.log 2>&1
for n in 4 296; do
    RECON_B200_LIB=$PWD/paper_2504_06182_b200/lib/librecon_b200_prof.so timeout 600 python tools/batch_prof.py c5 $n > $O/phase_c5_$n.txt 2>&1
done
bash tools/checked_run.sh $O/checked > $O/checked_run.log 2>&1; echo "checked rc=$?"
echo done

#!/bin/bash
# Round-2 profile refresh on one B200 (run under gpurun; results in gpurun_out/prof_r02):
#  1. the bench's launch list (gpu__time_duration, clocks not locked)
#  2. ncu --set full of the C5 pipeline kernels at 64 instances (a 1,024-instance
#     capture would have ncu save/restore ~100 GB of device memory per replay)
#  3. ncu --set full of the C3 pipeline batching kernel
#  4. the clock64 phase breakdown of the batching kernels (-DRECON_BATCH_PROF build)
cd "$(dirname "$0")/.."
O=gpurun_out/prof_r02
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-extras --no-cpu > $O/bench_under_ncu.log 2>&1; echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"batch_pipeline_kernel|batch_wide|pl_walk_warp|bird_kernel|pl_mark2" -c 6 \
    -o $O/c5_full -f python tools/perf_probe.py c5_pipeline_64 > $O/ncu_c5.log 2>&1; echo "c5 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"batch_pipeline_kernel|pl_dag_small" -c 3 \
    -o $O/c3_full -f python tools/perf_probe.py c3_pipeline_none > $O/ncu_c3.log 2>&1; echo "c3 full rc=$?"
# text summaries only (gpurun copies back at most 64 MiB): metrics + stalls per
# kernel, and the hottest source lines per kernel
for r in c5_full c3_full; do
    python tools/ncu_raw.py $O/$r.ncu-rep > $O/${r}_raw.txt 2>&1
done
for k in batch_pipeline_kernel batch_wide pl_walk_warp_kernel.0 pl_walk_warp_kernel.1 bird_kernel; do
    ncu -i $O/c5_full.ncu-rep --page source --csv --print-source cuda,sass -k regex:"$k" > $O/src.csv 2>/dev/null
    python tools/ncu_lines.py $O/src.csv 30 > $O/c5_lines_${k//[^a-z0-9_]/_}.txt 2>&1
done
ncu -i $O/c3_full.ncu-rep --page source --csv --print-source cuda,sass -k regex:batch_pipeline_kernel > $O/src.csv 2>/dev/null
python tools/ncu_lines.py $O/src.csv 30 > $O/c3_lines_batch_pipeline_kernel.txt 2>&1
rm -f $O/src.csv $O/*.ncu-rep
touch paper_2504_06182_b200/csrc/batching.cu paper_2504_06182_b200/csrc/batch_wide.cu
RECON_BUILD_TAG=prof RECON_NVCC_EXTRA=-DRECON_BATCH_PROF python paper_2504_06182_b200/build_native.py > $O/prof_build.log 2>&1
for n in 4 512; do
    RECON_B200_LIB=$PWD/paper_2504_06182_b200/lib/librecon_b200_prof.so timeout 600 python tools/batch_prof.py c5 $n > $O/phase_c5_$n.txt 2>&1
done
echo done

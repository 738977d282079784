#!/bin/bash
# The checked build: every kernel compiled with -DRECON_CHECKED (device-side
# invariant checks that print and trap, common.cuh RB_CHECK) and -G-free
# -lineinfo, into paper_2504_06182_b200/lib/librecon_b200_checked.so; then
# every kernel family (tools/sanitize_cases.py, each result compared with
# the oracle) and the scale parity suite run against it.  This stands in for
# compute-sanitizer, which is closed on this GPU pool.
#   bash tools/checked_run.sh [outdir]
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/checked}
mkdir -p "$OUT"
RECON_BUILD_TAG=checked RECON_NVCC_EXTRA="-DRECON_CHECKED" python paper_2504_06182_b200/build_native.py > "$OUT/build.log" 2>&1 || { echo "checked build failed"; tail "$OUT/build.log"; exit 1; }
export RECON_B200_LIB=$PWD/paper_2504_06182_b200/lib/librecon_b200_checked.so
: > "$OUT/summary.txt"
for FAM in solves chains pipeline stats validators wire sim; do
    timeout 900 python tools/sanitize_cases.py $FAM > "$OUT/$FAM.log" 2>&1; echo "$FAM rc=$?" | tee -a "$OUT/summary.txt"
done
RECON_BATCH_WIDE=1 timeout 900 python tools/sanitize_cases.py pipeline > "$OUT/pipeline_wide.log" 2>&1; echo "pipeline (wide forced) rc=$?" | tee -a "$OUT/summary.txt"
RECON_BATCH_LEAP=0 timeout 900 python tools/sanitize_cases.py pipeline > "$OUT/pipeline_noleap.log" 2>&1; echo "pipeline (leap off) rc=$?" | tee -a "$OUT/summary.txt"
RECON_BATCH_LEAP=2 timeout 900 python tools/sanitize_cases.py pipeline > "$OUT/pipeline_leap.log" 2>&1; echo "pipeline (leap forced on small grids) rc=$?" | tee -a "$OUT/summary.txt"
timeout 1800 python -m pytest tests/test_batching_scale_gpu.py tests/test_batching_gpu.py tests/test_grid_gpu.py -q -x > "$OUT/pytest.log" 2>&1; echo "pytest scale+batching+grid (checked lib) rc=$?: $(tail -1 $OUT/pytest.log)" | tee -a "$OUT/summary.txt"
grep -h "RB_CHECK failed" "$OUT"/*.log | sort | uniq -c | tee -a "$OUT/summary.txt"
echo "RB_CHECK failures: $(grep -h 'RB_CHECK failed' "$OUT"/*.log | wc -l)" | tee -a "$OUT/summary.txt"

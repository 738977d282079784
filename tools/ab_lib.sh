# A/B of two builds of the native library on one box: exp/head.so (A) vs the working tree (B)
# usage: CASES="c3_pipeline_none c4_pipeline_redrec_64" bash tools/ab_lib.sh
for r in 1 2; do
  echo "A"; RECON_B200_LIB=$PWD/exp/head.so python tools/perf_probe.py $CASES | cut -c1-90
  echo "B"; python tools/perf_probe.py $CASES | cut -c1-90
done

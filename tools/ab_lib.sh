# A/B of two builds of the native library on one box: exp/head.so (A) vs the working tree (B)
# usage: CASES="c3_pipeline_none c4_pipeline_redrec_64" bash tools/ab_lib.sh
short() { python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith('{'): continue
    for k,v in json.loads(l).items():
        print(k, ' '.join(f'{x}={v[x]:.4g}' for x in ('ms','plan_ms','exec_ms') if x in v))
"; }
for r in 1 2; do
  echo "A"; RECON_B200_LIB=$PWD/exp/head.so python tools/perf_probe.py $CASES | short
  echo "B"; python tools/perf_probe.py $CASES | short
done

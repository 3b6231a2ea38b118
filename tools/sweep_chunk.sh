#!/bin/bash
# Sweep the chunk kernel's consumer groups / ring stages on the headline
# decode workload (bench.py --no-rows).  Usage: bash tools/sweep_chunk.sh tag
TAG=${1:-sweep}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for cfg in ${SWEEP:-"0 0" "2 8" "4 8" "8 8" "4 4" "5 10" "2 4"}; do
  set -- $cfg
  LABUF_CHUNK_NG=$1 LABUF_CHUNK_NS=$2 timeout 300 python bench.py --no-rows --no-cpu --steps 20 --warmup 3 > $OUT/b_$1_$2.json 2>$OUT/b_$1_$2.err
  python - $OUT/b_$1_$2.json "$1 $2" <<'PY' >> $OUT/summary.txt
import json,sys
try:
    d=json.load(open(sys.argv[1]))
    k=d["kernels"]
    print(sys.argv[2], "decode_us %.2f gbs %.0f | flush_us %.1f | rec_us %.2f | us/tok %.2f speedup %.3f" % (k["decode"]["us_per_launch"], k["decode"]["gbs"], k["flush"]["us_per_launch"], k["recurrent_step"]["us_per_launch"], d["us_per_token"], d["speedup_vs_recurrent"]))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
cat $OUT/summary.txt

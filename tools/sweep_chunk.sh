#!/bin/bash
# Sweep chunk-kernel tuning knobs on the headline decode workload
# (bench.py --no-rows).  Usage: SWEEP="A=1,B=2 C=3 ..." bash tools/sweep_chunk.sh tag
# Each sweep item is a comma-separated list of environment assignments.
TAG=${1:-sweep}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for cfg in ${SWEEP:-LABUF_CHUNK_RING=1}; do
  envs=$(echo "$cfg" | tr ',' ' ')
  env $envs timeout 300 python bench.py --no-rows --no-cpu --steps 20 --warmup 3 > $OUT/b_$cfg.json 2>$OUT/b_$cfg.err
  python - $OUT/b_$cfg.json "$cfg" <<'PY' >> $OUT/summary.txt
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

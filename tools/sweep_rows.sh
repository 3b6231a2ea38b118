#!/bin/bash
# Sweep knobs on the verify / direct rows (bench.py rows).  Usage: SWEEP="A=1,B=2 ..." bash tools/sweep_rows.sh tag
TAG=${1:-rows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for cfg in ${SWEEP:-X=0}; do
  envs=$(echo "$cfg" | tr ',' ' ')
  env $envs timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 > $OUT/b_$cfg.json 2>$OUT/b_$cfg.err
  python - $OUT/b_$cfg.json "$cfg" <<'PY' >> $OUT/summary.txt
import json,sys
try:
    d=json.load(open(sys.argv[1])); r=d["rows"]; v=r["verify_commit"]; x=r["direct"]
    print(sys.argv[2], "decode %.2f flush %.1f | verify %.1f commit %.1f (rec %.1f) | direct %.1f (rec %.1f)" % (d["kernels"]["decode"]["us_per_launch"], d["kernels"]["flush"]["us_per_launch"], v["verify_us"], v["commit_us"], v["recurrent_us_per_round"], x["us_per_step"], x["recurrent_us_per_step"]))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
cat $OUT/summary.txt

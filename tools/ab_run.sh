#!/bin/bash
# A/B/... several library builds on ONE GPU box (box-to-box variance is 2-5 %).
# On the box:  bash tools/ab_run.sh tag "A B C" rounds [bench flags...]
# runs bench.py with LABUF_LIB=ab/liblabuf_<v>.so alternately, summary in gpurun_out/<tag>/summary.txt
TAG=$1; VARS=$2; ROUNDS=${3:-2}; shift 3
OUT=gpurun_out/$TAG
mkdir -p $OUT
for r in $(seq 1 $ROUNDS); do
  for v in $VARS; do
    LABUF_LIB=$PWD/ab/liblabuf_$v.so timeout 300 python bench.py --no-cpu --no-e2e --no-config5 --no-config1 "$@" > $OUT/$v$r.json 2>$OUT/$v$r.err || true
    python - $OUT/$v$r.json "$v$r" <<'PY' >> $OUT/summary.txt
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["kernels"]; r=d.get("rows",{}); v=r.get("verify_commit",{}); x=r.get("direct",{}); m=r.get("flush_mode_ii",{}); pf=r.get("prefill",{})
    print(sys.argv[2], "decode %.2f flush %.1f rec %.2f | us/tok %.2f | verify %.1f commit %.1f | direct %.1f | raw %.1f | prefill %.0f us" % (k["decode"]["us_per_launch"], k["flush"]["us_per_launch"], k["recurrent_step"]["us_per_launch"], d["us_per_token"], v.get("verify_us",0), v.get("commit_us",0), x.get("us_per_step",0), m.get("us_per_launch",0), 1e3 * pf.get("ms", 0)))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
  done
done
cat $OUT/summary.txt

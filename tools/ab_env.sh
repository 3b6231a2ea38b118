#!/bin/bash
# A/B of one library build under different environment settings, on ONE GPU box.
# On the box:  bash tools/ab_env.sh tag VAR "a b" rounds [bench flags...]
# runs bench.py with VAR=a, VAR=b alternately ("unset": VAR removed); summary in gpurun_out/<tag>/summary.txt
TAG=$1; VAR=$2; VALS=$3; ROUNDS=${4:-2}; shift 4
OUT=gpurun_out/$TAG
mkdir -p $OUT
for r in $(seq 1 $ROUNDS); do
  for v in $VALS; do
    if [ "$v" = unset ]; then E="env -u $VAR"; else E="env $VAR=$v"; fi
    $E timeout 400 python bench.py --no-cpu --no-e2e --no-config1 "$@" > $OUT/$v$r.json 2>$OUT/$v$r.err || true
    python - $OUT/$v$r.json "$v$r" <<'PY' >> $OUT/summary.txt
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["kernels"]; r=d.get("rows",{}); v=r.get("verify_commit",{}); x=r.get("direct",{}); pf=r.get("prefill",{}); c5=r.get("config5",{})
    print(sys.argv[2], "decode %.2f flush %.1f | us/tok %.2f | verify %.1f commit %.1f | direct %.1f | prefill %.0f us | config5 %s" % (k["decode"]["us_per_launch"], k["flush"]["us_per_launch"], d["us_per_token"], v.get("verify_us",0), v.get("commit_us",0), x.get("us_per_step",0), 1e3 * pf.get("ms", 0), json.dumps({kk: c5[kk] for kk in c5 if "ms" in kk or "us" in kk})))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
  done
done
cat $OUT/summary.txt

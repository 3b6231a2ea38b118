#!/bin/bash
# A/B two library builds on ONE GPU box (box-to-box variance is 5-10%).
# Here:   bash tools/ab.sh prepare   -> builds HEAD into /root/repo/ab/liblabuf_A.so and the
#                                        working tree into ab/liblabuf_B.so
# On box: bash tools/ab.sh run tag [rounds]  -> alternates A, B bench runs, summary in gpurun_out/tag
set -e
cmd=$1
if [ "$cmd" = prepare ]; then
  mkdir -p ab
  python -m paper_2605_19049_b200.build --force >/dev/null && cp paper_2605_19049_b200/liblabuf.so ab/liblabuf_B.so
  git stash -q
  python -m paper_2605_19049_b200.build --force >/dev/null && cp paper_2605_19049_b200/liblabuf.so ab/liblabuf_A.so
  git stash pop -q
  python -m paper_2605_19049_b200.build --force >/dev/null
  ls -la ab
  exit 0
fi
TAG=${2:-ab}
ROUNDS=${3:-2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for r in $(seq 1 $ROUNDS); do
  for v in A B; do
    LABUF_LIB=$PWD/ab/liblabuf_$v.so timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 > $OUT/$v$r.json 2>$OUT/$v$r.err || true
    python - $OUT/$v$r.json "$v$r" <<'PY' >> $OUT/summary.txt
import json,sys
try:
    d=json.load(open(sys.argv[1])); k=d["kernels"]; r=d.get("rows",{}); v=r.get("verify_commit",{}); x=r.get("direct",{})
    print(sys.argv[2], "decode %.2f flush %.1f rec %.2f | us/tok %.2f | verify %.1f commit %.1f | direct %.1f" % (k["decode"]["us_per_launch"], k["flush"]["us_per_launch"], k["recurrent_step"]["us_per_launch"], d["us_per_token"], v.get("verify_us",0), v.get("commit_us",0), x.get("us_per_step",0)))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
  done
done
cat $OUT/summary.txt

#!/bin/bash
# Config-2 sweeps (BASELINE configs[1], the Fig. 4
# analogue): buffer size C at batch 64, and batch at C = 16, each with the
# in-run recurrent baseline.  Writes gpurun_out/$1/sweep.jsonl + summary.txt.
TAG=${1:-sweep_c2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
run() {  # batch chunk layers
  timeout 600 python bench.py --no-rows --no-cpu --no-e2e --no-config1 --no-config5 --steps 10 --warmup 3 \
      --batch $1 --chunk $2 --layers $3 > $OUT/b_$1_$2.json 2> $OUT/b_$1_$2.err
  python - $OUT/b_$1_$2.json $1 $2 <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k = d["kernels"]
    row = {"batch": int(sys.argv[2]), "chunk": int(sys.argv[3]), "us_per_token": d["us_per_token"],
           "recurrent_us_per_token": d["recurrent"]["us_per_token"], "speedup": d["speedup_vs_recurrent"],
           "latency_reduction_pct": d["latency_reduction_pct_vs_recurrent"],
           "decode_us": k["decode"]["us_per_launch"], "decode_frac": k["decode"]["frac_of_measured"],
           "flush_us": k["flush"]["us_per_launch"], "hbm_frac_of_measured": d["hbm_frac_of_measured"]}
    print(json.dumps(row))
except Exception as e:
    print(json.dumps({"batch": sys.argv[2], "chunk": sys.argv[3], "failed": str(e)}))
PY
}
for C in 1 8 16 22 32; do run 64 $C 8; done
for B in 1 8 256 1024; do run $B 16 $([ $B -ge 256 ] && echo 4 || echo 8); done
cat $OUT/summary.txt

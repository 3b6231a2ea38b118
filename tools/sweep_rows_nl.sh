#!/bin/bash
# Config-3 draft sweep (Fig. 5 analogue) and config-4 context sweep (Fig. 7
# analogue), each against the in-run recurrent kernels.  -> gpurun_out/$1/summary.txt
TAG=${1:-sweep_rows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for N in 1 2 4 8; do
  timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 --drafts $N --direct-l0 64 > $OUT/n$N.json 2>$OUT/n$N.err
  python -c "import json,sys; d=json.load(open('$OUT/n$N.json')); v=d['rows']['verify_commit']; print(json.dumps({'drafts': $N, 'verify_us': v['verify_us'], 'commit_us': v['commit_us'], 'round_us': v['us_per_round'], 'recurrent_round_us': v['recurrent_us_per_round'], 'speedup': v['speedup_vs_recurrent'], 'verify_frac': v['verify_frac_of_measured']}))" >> $OUT/summary.txt
done
for L0 in 16 32 96; do
  timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 --direct-l0 $L0 > $OUT/l$L0.json 2>$OUT/l$L0.err
  python -c "import json,sys; d=json.load(open('$OUT/l$L0.json')); x=d['rows']['direct']; print(json.dumps({'l0': $L0, 'direct_us': x['us_per_step'], 'recurrent_us': x['recurrent_us_per_step'], 'speedup': x['speedup_vs_recurrent'], 'frac': x['frac_of_measured']}))" >> $OUT/summary.txt
done
cat $OUT/summary.txt

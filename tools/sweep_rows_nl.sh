#!/bin/bash
# Config-3 draft sweep (Fig. 5 analogue) against the in-run recurrent verify
# + copy, and the multi-round (append) variant.  -> gpurun_out/$1/summary.txt
# (the config-4 context sweep, Fig. 7 analogue, is part of every bench line:
#  rows.direct.fig7)
TAG=${1:-sweep_rows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for N in 1 2 4 8 16; do
  timeout 600 python bench.py --no-cpu --no-e2e --no-config1 --no-config5 --steps 10 --warmup 3 --drafts $N > $OUT/n$N.json 2>$OUT/n$N.err
  python -c "import json,sys; d=json.loads(open('$OUT/n$N.json').read().strip().splitlines()[-1]); v=d['rows']['verify_commit']; print(json.dumps({'drafts': $N, 'verify_us': v['verify_us'], 'commit_us': v['commit_us'], 'round_us': v['us_per_round'], 'recurrent_round_us': v['recurrent_us_per_round'], 'speedup': v['speedup_vs_recurrent'], 'verify_frac': v['verify_frac_of_measured'], 'multi_round_us': v['multi_round']['us_per_round'], 'multi_round_speedup': v['multi_round']['speedup_vs_recurrent']}))" >> $OUT/summary.txt
done
cat $OUT/summary.txt

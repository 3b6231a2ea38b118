#!/bin/bash
# compute-sanitizer pass over the small hot-path invocation of
# __graft_entry__.smoke() (prefill, decode cycle + tcgen05 flush, 4-draft
# verify + commit, direct step), a paged mixed-batch step and the mode-ii
# flush driver tools/run_raw_small.py (run under gpurun).
OUT=gpurun_out/${1:-sanitize}
mkdir -p $OUT
PY="import sys; sys.path.insert(0, '.'); import __graft_entry__ as g; g.smoke()"
for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "$PY" > $OUT/$tool.log 2>&1
    echo "$tool rc=$?" >> $OUT/summary.txt
    tail -3 $OUT/$tool.log >> $OUT/summary.txt
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/run_mixed.py > $OUT/memcheck_mixed.log 2>&1
echo "memcheck mixed rc=$?" >> $OUT/summary.txt
tail -3 $OUT/memcheck_mixed.log >> $OUT/summary.txt
# flush mode ii (fold_ut.cu): multi-chunk fold and direct-slot compression, bf16 and fp32
for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/run_raw_small.py > $OUT/${tool}_raw.log 2>&1
    echo "$tool raw rc=$?" >> $OUT/summary.txt
    tail -3 $OUT/${tool}_raw.log >> $OUT/summary.txt
done
cat $OUT/summary.txt

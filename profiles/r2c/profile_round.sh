#!/bin/bash
# Round profiling pass (run under gpurun): the launch list of the bench step
# and one `ncu --set full` capture per hot-path kernel, into gpurun_out/$1/.
set -x
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches.csv \
    -k regex:'chunk_|fold_|recurrent_|stage_' python bench.py --steps 2 --warmup 3 --no-cpu --no-rows --no-e2e > $OUT/launches.log 2>&1
FULL="$NCU --set full --import-source on"
$FULL -k regex:chunk_cta -s 8 -c 1 -o $OUT/decode python tools/run_decode.py 1 > $OUT/decode.log 2>&1
$FULL -k regex:fold -c 1 -o $OUT/flush python tools/run_decode.py 1 > $OUT/flush.log 2>&1
$FULL -k regex:recurrent_step -s 4 -c 1 -o $OUT/recurrent_step python tools/run_decode.py 1 > $OUT/rec.log 2>&1
$FULL -k regex:chunk_cta -s 1 -c 1 -o $OUT/verify python tools/run_rows.py verify 2 > $OUT/verify.log 2>&1
$FULL -k regex:fold -s 1 -c 1 -o $OUT/commit python tools/run_rows.py verify 2 > $OUT/commit.log 2>&1
$FULL -k regex:recurrent_verify -s 1 -c 1 -o $OUT/recurrent_verify python tools/run_rows.py rverify 2 > $OUT/rverify.log 2>&1
$FULL -k regex:chunk_cta -s 5 -c 1 -o $OUT/direct python tools/run_rows.py direct 3 > $OUT/direct.log 2>&1
$FULL -k regex:fold -s 1 -c 1 -o $OUT/flush_raw python tools/run_raw_flush.py 2 > $OUT/flush_raw.log 2>&1
$FULL -k regex:chunk_cta -s 3 -c 1 -o $OUT/prefill python tools/run_prefill.py > $OUT/prefill.log 2>&1
ls -la $OUT
# summaries on the box (reports > 8 MB stay behind: gpurun copies back <= 64 MiB)
python tools/launch_summary.py $OUT/launches.csv > $OUT/ncu_launches_summary.csv
python tools/ncu_traffic.py $OUT decode=$OUT/decode.ncu-rep flush=$OUT/flush.ncu-rep \
    recurrent_step=$OUT/recurrent_step.ncu-rep verify=$OUT/verify.ncu-rep commit=$OUT/commit.ncu-rep \
    recurrent_verify=$OUT/recurrent_verify.ncu-rep direct=$OUT/direct.ncu-rep flush_raw=$OUT/flush_raw.ncu-rep \
    prefill=$OUT/prefill.ncu-rep > $OUT/traffic.log 2>&1
for k in decode flush recurrent_step verify commit recurrent_verify direct flush_raw prefill; do
    python tools/ncu_summary.py $OUT/$k.ncu-rep --sass 12 > $OUT/ncu_${k}_stalls.txt 2>&1
    python tools/ncu_lines.py $OUT/$k.ncu-rep 20 > $OUT/ncu_${k}_lines.txt 2>&1
done
find $OUT -name '*.ncu-rep' -size +8M -delete
rm -f $OUT/launches.csv
ls -la $OUT

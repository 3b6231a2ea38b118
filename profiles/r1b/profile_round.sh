#!/bin/bash
# Round profiling pass (run under gpurun): launch list of the bench step and
# one `ncu --set full` capture per hot-path kernel, into gpurun_out/$1/.
set -x
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches.csv \
    -k regex:'chunk_|fold_|recurrent_' python bench.py --steps 2 --warmup 3 --no-cpu --no-rows > $OUT/launches.log 2>&1
FULL="$NCU --set full --import-source on"
$FULL -k regex:chunk_cta -s 8 -c 1 -o $OUT/decode python tools/run_decode.py 1 > $OUT/decode.log 2>&1
$FULL -k regex:chunk_cta -s 15 -c 1 -o $OUT/decode_fused_step python tools/run_decode.py 1 fused > $OUT/decode_fused.log 2>&1
# DRAM bytes of every launch of one fused cycle (metrics only: cheap)
$NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:chunk_cta -c 16 \
    -o $OUT/decode_cycle_fused python tools/run_decode.py 1 fused > $OUT/decode_cycle.log 2>&1
$FULL -k regex:fold -c 1 -o $OUT/flush python tools/run_decode.py 1 > $OUT/flush.log 2>&1
$FULL -k regex:recurrent_step -s 4 -c 1 -o $OUT/recurrent_step python tools/run_decode.py 1 > $OUT/rec.log 2>&1
$FULL -k regex:chunk_cta -s 1 -c 1 -o $OUT/verify python tools/run_rows.py verify 2 > $OUT/verify.log 2>&1
$FULL -k regex:fold -s 1 -c 1 -o $OUT/commit python tools/run_rows.py verify 2 > $OUT/commit.log 2>&1
$FULL -k regex:chunk_cta -s 5 -c 1 -o $OUT/direct python tools/run_rows.py direct 3 > $OUT/direct.log 2>&1
$FULL -k regex:fold -s 1 -c 1 -o $OUT/flush_raw python tools/run_raw_flush.py 2 > $OUT/flush_raw.log 2>&1
ls -la $OUT
# summaries on the box (reports > 8 MB stay behind: gpurun copies back <= 64 MiB)
python tools/launch_summary.py $OUT/launches.csv > $OUT/ncu_launches_summary.csv
python tools/ncu_traffic.py $OUT decode=$OUT/decode.ncu-rep decode_cycle_fused=$OUT/decode_cycle_fused.ncu-rep \
    decode_fused_step=$OUT/decode_fused_step.ncu-rep flush=$OUT/flush.ncu-rep \
    recurrent_step=$OUT/recurrent_step.ncu-rep verify=$OUT/verify.ncu-rep commit=$OUT/commit.ncu-rep \
    direct=$OUT/direct.ncu-rep flush_raw=$OUT/flush_raw.ncu-rep > $OUT/traffic.log 2>&1
for k in decode decode_fused_step flush recurrent_step verify commit direct flush_raw; do
    python tools/ncu_summary.py $OUT/$k.ncu-rep --sass 12 > $OUT/ncu_${k}_stalls.txt 2>&1
done
find $OUT -name '*.ncu-rep' -size +8M -delete
rm -f $OUT/launches.csv
ls -la $OUT

#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, ncu launch list and full
# captures of the top kernels.  Usage (from the repo root, under gpurun):
#   bash tools/gpu_check.sh [tag]
# Everything lands in gpurun_out/<tag>/.
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'chunk_|fold_|recurrent_|decode_' -c 3000 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/ncu_launch_bench.log 2>&1
for K in chunk_cta fold_kernel recurrent_step_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
      -o $OUT/prof_$K python bench.py --steps 2 --warmup 3 --no-rows --no-cpu > $OUT/ncu_$K.log 2>&1
done
python tools/ncu_traffic.py $OUT decode=$OUT/prof_chunk_cta.ncu-rep flush=$OUT/prof_fold_kernel.ncu-rep \
    recurrent_step=$OUT/prof_recurrent_step_kernel.ncu-rep > $OUT/ncu_traffic.log 2>&1
fi
ls -la $OUT

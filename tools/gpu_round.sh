#!/bin/bash
# One GPU round: smoke, GPU parity tests, 1-GPU bench, ncu launch list + full capture.
# Usage (from the dev container): gpurun --timeout 1500 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv >> $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python tools/bench_paths.py > $OUT/paths.jsonl 2> $OUT/paths.err; echo "paths rc=$?" >> $OUT/paths.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_launch_bench.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather -s 3 -c 1 -o $OUT/prof_gather \
      python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_full.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:plan_canon -s 3 -c 1 -o $OUT/prof_plan \
      python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_full_plan.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_pipe -s 3 -c 1 -o $OUT/prof_dense \
      python tools/bench_paths.py --only cfg3 --reps 2 > $OUT/ncu_full_dense.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_pipe -s 3 -c 1 -o $OUT/prof_dense_cfg2 \
      python tools/bench_paths.py --only cfg2d --reps 2 > $OUT/ncu_full_dense_cfg2.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:oae_warp -s 3 -c 1 -o $OUT/prof_oae \
      python tools/bench_paths.py --only cfg4 --reps 2 > $OUT/ncu_full_oae.log 2>&1
fi
echo done > $OUT/done

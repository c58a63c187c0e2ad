#!/bin/bash
# One GPU round: smoke, GPU parity tests, the reference's own tests through the
# drop-in, 1-GPU bench (with its sparse4d block), optional ncu captures.
# Usage (from the dev container): gpurun --timeout 2400 -- 'bash tools/gpu_round.sh <tag>'
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv >> $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 900 python tools/run_reference_tests.py > $OUT/reference_tests.log 2>&1; echo "rc=$?" >> $OUT/reference_tests.log
  DROPIN_ALL=1 timeout 900 python tools/run_reference_tests.py test_features.py test_bench.py test_oae.py \
      "test_acceptance.py::test_criterion_1_msda_parity" > $OUT/reference_tests_all.log 2>&1; echo "rc=$?" >> $OUT/reference_tests_all.log
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
fi
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 --no-sparse4d > $OUT/ncu_launch_bench.log 2>&1
fi
echo done > $OUT/done

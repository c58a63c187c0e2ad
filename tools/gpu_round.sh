#!/bin/bash
# One GPU round: smoke, GPU parity tests, the reference's own tests through the
# drop-in, 1-GPU bench (with its sparse4d block), ncu launch list + captures.
# Usage (from the dev container): gpurun --timeout 3000 -- 'bash tools/gpu_round.sh <tag>'
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv >> $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 900 python tools/run_reference_tests.py > $OUT/reference_tests.log 2>&1; echo "rc=$?" >> $OUT/reference_tests.log
  DROPIN_ALL=1 timeout 900 python tools/run_reference_tests.py test_features.py test_bench.py test_oae.py \
      "test_acceptance.py::test_criterion_1_msda_parity" > $OUT/reference_tests_all.log 2>&1; echo "rc=$?" >> $OUT/reference_tests_all.log
  # the unmodified reference's own criterion 2 on this host (its scalar msda_reference sets the runtime)
  (cd baseline/_ref_tests && PYTHONPATH=../_ref PYTHONDONTWRITEBYTECODE=1 timeout 600 python -m pytest -p no:cacheprovider -q \
      "test_acceptance.py::test_criterion_2_msda_throughput" > ../../$OUT/reference_unmodified_crit2.log 2>&1; echo "rc=$?" >> ../../$OUT/reference_unmodified_crit2.log)
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
  timeout 600 python bench.py --config cfg5-stream --steps 10 --warmup 3 > $OUT/bench_cfg5_stream.json 2>&1
  timeout 600 python bench.py --config cfg5-camera --steps 10 --warmup 3 > $OUT/bench_cfg5_camera.json 2>&1
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 --no-sparse4d > $OUT/ncu_launch_bench.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"staged|gather_pipe|dense_exact|normalize" -c 20 --csv --log-file $OUT/launches_cfg3.csv \
      python tools/dev_one.py 64 float16 fast_h2 3 > $OUT/ncu_launch_cfg3.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_pipe -s 3 -c 1 -o $OUT/prof_gather \
      python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --no-sparse4d > $OUT/ncu_full.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"staged|gather_pipe" -s 2 -c 2 -o $OUT/prof_cfg3_h2 \
      python tools/dev_one.py 64 float16 fast_h2 2 > $OUT/ncu_full_cfg3.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dense_exact" -c 1 -o $OUT/prof_cfg3_exact \
      python tools/dev_one.py 64 float16 exact 1 > $OUT/ncu_full_cfg3x.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:oae_warp -s 3 -c 1 -o $OUT/prof_oae \
      python tools/bench_paths.py --only cfg4 --reps 2 > $OUT/ncu_full_oae.log 2>&1
fi
echo done > $OUT/done

OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_csr.py tests/test_gpu_dense.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/bench.json 2> $OUT/bench.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:plan_canon -s 3 -c 1 -o $OUT/prof_plan python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1

OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_csr.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for c in 1 2 4; do MSDA_CSR_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done

OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_dense.py tests/test_gpu_scene.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python tools/bench_paths.py --only cfg1d,cfg3,cfg3_h2,cfg4d,cfg5,cfg2d > $OUT/paths_cb.jsonl 2>&1
MSDA_DENSE_KERNEL=warpcam timeout 300 python tools/bench_paths.py --only cfg1d,cfg3,cfg3_h2,cfg4d,cfg2d > $OUT/paths_wc.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:camblk -s 2 -c 1 -o $OUT/prof_cb python tools/bench_paths.py --only cfg3 --reps 2 > /dev/null 2>&1

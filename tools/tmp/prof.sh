OUT=gpurun_out/$1; mkdir -p $OUT
N="ncu --set full --clock-control none --import-source on"
timeout 300 $N -k regex:oae -s 2 -c 1 -o $OUT/prof_oae python tools/bench_paths.py --only cfg4 --reps 2 > /dev/null 2>&1
timeout 300 $N -k regex:paint_kernel -s 2 -c 1 -o $OUT/prof_paint python tools/bench_paths.py --only paint --reps 2 > /dev/null 2>&1
timeout 300 $N -k regex:assoc -s 2 -c 1 -o $OUT/prof_assoc python tools/bench_paths.py --only assoc --reps 2 > /dev/null 2>&1
timeout 300 $N -k regex:dense_canon -s 2 -c 1 -o $OUT/prof_dense_canon python tools/bench_paths.py --only cfg1d_exact --reps 2 > /dev/null 2>&1
timeout 300 $N -k regex:gather_pipe -s 2 -c 1 -o $OUT/prof_dense_exact_gather python tools/bench_paths.py --only cfg1d_exact --reps 2 > /dev/null 2>&1
timeout 300 $N -k regex:warpcam -s 2 -c 1 -o $OUT/prof_dense_cfg4 python tools/bench_paths.py --only cfg4d --reps 2 > /dev/null 2>&1

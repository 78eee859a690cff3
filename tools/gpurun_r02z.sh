cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02z2; mkdir -p $OUT
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 1500 python tools/sweep.py > $OUT/sweep_c5.jsonl 2> $OUT/sweep_c5.err

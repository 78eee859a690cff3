cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02bu; mkdir -p $OUT
for i in 1 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_on_$i.json 2> $OUT/bench_on_$i.err
  RK_ATTN_DECODE=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_off_$i.json 2> $OUT/bench_off_$i.err
done
timeout 600 python tools/capture_bench.py c2 256 > $OUT/capture_c2_on.json 2>&1
RK_ATTN_DECODE=0 timeout 600 python tools/capture_bench.py c2 256 > $OUT/capture_c2_off.json 2>&1

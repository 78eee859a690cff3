cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02m; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > $OUT/pytest_attn.log 2>&1; echo "exit $?" >> $OUT/pytest_attn.log
RK_ATTN_MERGE=0 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > $OUT/pytest_attn_merge0.log 2>&1; echo "exit $?" >> $OUT/pytest_attn_merge0.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
for cfg in "X=0" "RK_ATTN_MERGE=0" "RK_ATTN_SPLITWAVES=100" "RK_ATTN_SPLITWAVES=100,RK_ATTN_SPLITDIV=1" "RK_ATTN_SPLITWAVES=100,RK_ATTN_SPLITDIV=3" "RK_ATTN_SPLITWAVES=100,RK_ATTN_SPLITDIV=3,RK_ATTN_MINPART=2" "RK_ATTN_SPLITWAVES=100,RK_ATTN_SPLITDIV=4,RK_ATTN_MINPART=2"; do
  env $(echo $cfg | tr ',' ' ') timeout 300 $B > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
done

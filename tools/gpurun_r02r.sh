cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > $OUT/pytest_attn.log 2>&1; echo "exit $?" >> $OUT/pytest_attn.log
for cfg in "X=0" "RK_ATTN_MERGE=0" "RK_ATTN_SPLITWAVES=100" "RK_ATTN_MINPART=2" "RK_ATTN_SPLITWAVES=100,RK_ATTN_SPLITDIV=1"; do
  echo "== $cfg" >> $OUT/mb.txt
  env $(echo $cfg | tr ',' ' ') timeout 120 python tools/microbench.py rows >> $OUT/mb.txt 2>&1
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off > $OUT/bench.json 2> $OUT/bench.err

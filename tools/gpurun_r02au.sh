cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02au; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for cfg in "X=0" "RK_ATTN_PTMEM=0"; do
  echo "== $cfg" >> $OUT/mb.txt
  env $(echo $cfg | tr ',' ' ') timeout 120 python tools/microbench.py rows >> $OUT/mb.txt 2>&1
  env $(echo $cfg | tr ',' ' ') timeout 200 python tools/microbench.py attn >> $OUT/mb.txt 2>&1
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off > $OUT/bench.json 2> $OUT/bench.err

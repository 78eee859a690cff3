cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02p2; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
for cfg in "X=0" "RK_ATTN_POLY=0xAA" "RK_ATTN_POLY=0x92" "RK_ATTN_POLY=0" "X=1"; do
  env $(echo $cfg | tr ',' ' ') timeout 300 $B > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
done

cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02l; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention or fixup" > $OUT/pytest_attn.log 2>&1; echo "exit $?" >> $OUT/pytest_attn.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
timeout 300 $B > $OUT/bench_pack1.json 2> $OUT/bench_pack1.err
RK_ATTN_PACK=0 timeout 300 $B > $OUT/bench_pack0.json 2> $OUT/bench_pack0.err
timeout 300 python tools/microbench.py attn > $OUT/microbench.txt 2>&1
RK_ATTN_PACK=0 timeout 300 python tools/microbench.py attn > $OUT/microbench_pack0.txt 2>&1

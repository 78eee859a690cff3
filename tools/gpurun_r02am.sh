cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02am; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py tests/test_gpu_wide.py tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 120 python tools/gemm_trace.py 320 16384 2048 2 > $OUT/trace_swap.txt 2>&1
timeout 300 python tools/microbench.py gemm > $OUT/mb.txt 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
timeout 300 $B > $OUT/bench.json 2> $OUT/bench.err
timeout 300 $B > $OUT/bench2.json 2> $OUT/bench2.err

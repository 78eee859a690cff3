cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02at; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
RK_GEMM_LOG=1 timeout 300 $B > $OUT/bench.json 2> $OUT/bench.err
timeout 300 $B > $OUT/bench2.json 2> $OUT/bench2.err

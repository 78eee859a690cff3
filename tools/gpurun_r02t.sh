cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02t; mkdir -p $OUT
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
RK_GEMM_LOG=1 timeout 300 $B > $OUT/bench.json 2> $OUT/bench.err
timeout 300 $B > $OUT/bench2.json 2> $OUT/bench2.err
RK_GEMM_OVERRIDE="4032d:3072:2048=128/2/1" timeout 300 $B > $OUT/bench_q128.json 2> $OUT/bench_q128.err
RK_GEMM_OVERRIDE="4032:3072:2048=128/2/1" timeout 300 $B > $OUT/bench_bq128.json 2> $OUT/bench_bq128.err
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log

cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02as; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 120 python tools/microbench.py rows > $OUT/mb.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off > $OUT/bench.json 2> $OUT/bench.err

cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02ab; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py -x -q -k "attention or bf16" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 120 python tools/microbench.py rows > $OUT/mb.txt 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
timeout 300 $B > $OUT/bench.json 2> $OUT/bench.err
timeout 300 $B > $OUT/bench2.json 2> $OUT/bench2.err

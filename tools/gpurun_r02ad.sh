cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02ad; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
timeout 300 $B > $OUT/bench.json 2> $OUT/bench.err
timeout 300 $B > $OUT/bench2.json 2> $OUT/bench2.err

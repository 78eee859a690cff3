cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02x; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_tc.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err

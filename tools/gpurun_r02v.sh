cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02v; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py -q -s > $OUT/pytest_tc.log 2>&1; echo "exit $?" >> $OUT/pytest_tc.log

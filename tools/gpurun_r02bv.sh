cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02bv; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_score.py tests/test_gpu_kernels.py -q -k "score or attention" > $OUT/pytest_k.log 2>&1; echo "exit $?" >> $OUT/pytest_k.log
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_$i.json 2> $OUT/bench_$i.err; done

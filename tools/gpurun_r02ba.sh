cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02ba; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_kernels.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_pf_$i.json 2> $OUT/bench_pf_$i.err
  RK_GEMM_DBG=4 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_nopf_$i.json 2> $OUT/bench_nopf_$i.err
done

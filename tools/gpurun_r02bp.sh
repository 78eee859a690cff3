cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02bq; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k attention > $OUT/pytest_attn.log 2>&1; echo "exit $?" >> $OUT/pytest_attn.log
python tools/microbench_m1.py > $OUT/m1.txt 2>&1
RK_ATTN_DECODE=0 python tools/microbench_m1.py > $OUT/m1_off.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_$i.json 2> $OUT/bench_$i.err; done
timeout 600 python tools/capture_bench.py c2 256 > $OUT/capture_c2.json 2>&1
RK_ATTN_DECODE=0 timeout 600 python tools/capture_bench.py c2 256 > $OUT/capture_c2_off.json 2>&1

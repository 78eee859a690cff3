cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02bi; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py tests/test_gpu_tc.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for s in "4032 2048 2048 1" "320 2048 2048 1" "1360 2048 8192 1"; do python tools/gemm_trace.py $s > "$OUT/trace_${s// /_}.txt" 2>&1; done
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_$i.json 2> $OUT/bench_$i.err; done

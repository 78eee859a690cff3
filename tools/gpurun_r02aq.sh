cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02aq; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py tests/test_gpu_wide.py tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for s in "4032 2048 2048 1" "1356 2048 8192 1"; do RK_BENCH_NORM=1 timeout 120 python tools/gemm_trace.py $s > "$OUT/trace_${s// /_}.txt" 2>&1; done
RK_BENCH_NORM=1 timeout 300 python tools/microbench.py gemm > $OUT/mb_norm.txt 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
timeout 300 $B > $OUT/bench.json 2> $OUT/bench.err
timeout 300 $B > $OUT/bench2.json 2> $OUT/bench2.err

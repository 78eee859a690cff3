cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02d; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "swap or gemm_store" -x -q > $OUT/pytest_swap.log 2>&1; echo "exit $?" >> $OUT/pytest_swap.log
timeout 900 python -m pytest tests/test_gpu_bf16.py -x -q -k swap > $OUT/pytest_swap_bf16.log 2>&1; echo "exit $?" >> $OUT/pytest_swap_bf16.log
timeout 900 python tools/gemm_sweep.py RK_GEMM_SWAP=0 RK_GEMM_SWAP=2 > $OUT/gemm_sweep.jsonl 2>&1
for sw in 0 1 2; do
  RK_GEMM_SWAP=$sw timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_swap$sw.json 2> $OUT/bench_swap$sw.err
done

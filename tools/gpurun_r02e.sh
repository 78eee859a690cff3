cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02e; mkdir -p $OUT
export SWEEP_SET=m320
timeout 600 python tools/gemm_sweep.py RK_GEMM_SWAP=0,RK_BENCH_COPIES=1 RK_GEMM_SWAP=2,RK_BENCH_COPIES=1 RK_GEMM_SWAP=0 RK_GEMM_SWAP=2 > $OUT/gemm_sweep_l2.jsonl 2>&1
export SWEEP_SET=c2
timeout 600 python tools/gemm_sweep.py RK_GEMM_ORDERED=0 RK_GEMM_ORDERED=1 > $OUT/gemm_sweep_ord.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "ordered or split" -x -q > $OUT/pytest_ord.log 2>&1; echo "exit $?" >> $OUT/pytest_ord.log
for o in 0 1; do RK_GEMM_SWAP=0 RK_GEMM_ORDERED=$o timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_ord$o.json 2> $OUT/bench_ord$o.err; done

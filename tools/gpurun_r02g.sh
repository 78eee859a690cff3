cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "swap" -x -q > $OUT/pytest_swap.log 2>&1; echo "exit $?" >> $OUT/pytest_swap.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -x -q > $OUT/pytest_parity.log 2>&1; echo "exit $?" >> $OUT/pytest_parity.log
timeout 900 python -m pytest tests/test_gpu_bf16.py -x -q -k swap > $OUT/pytest_swap_bf16.log 2>&1; echo "exit $?" >> $OUT/pytest_swap_bf16.log
SWEEP_SET=m320,c3 timeout 600 python tools/gemm_sweep.py RK_GEMM_SWAP=0 RK_GEMM_SWAP=2 > $OUT/gemm_sweep.jsonl 2>&1
for sw in 0 2; do RK_GEMM_SWAP=$sw timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_swap$sw.json 2> $OUT/bench_swap$sw.err; done
NV="--nvtx --nvtx-include relay_step/"
LEAN="python bench.py --steps 1 --warmup 0 --no-cpu --lean"
for spec in "realign_graft:0" "score_dh_kernel:0"; do
  pat=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu $NV --set full --import-source on --clock-control none -k regex:$pat -s $skip -c 1 -o $OUT/full_${pat}_$skip $LEAN > $OUT/ncu_${pat}_$skip.log 2>&1
done

OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > $OUT/pytest_kernels.log 2>&1; echo "exit $?" >> $OUT/pytest_kernels.log
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python tools/microbench.py attn > $OUT/micro_attn.log 2>&1
timeout 300 python tools/microbench.py gemm > $OUT/micro_gemm.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
echo done > $OUT/DONE

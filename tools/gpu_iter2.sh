OUT=gpurun_out/$1; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py -q > $OUT/k.log 2>&1
timeout 120 python tools/microbench.py attn > $OUT/m.log 2>&1
timeout 60 python tools/attn_trace.py > $OUT/trace.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err

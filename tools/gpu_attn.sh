# attention/gemm kernel tests, bf16 tests, microbenchmarks, one ncu capture of attn_kernel, bench
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q > $OUT/k.log 2>&1
timeout 300 python -m pytest tests/test_gpu_bf16.py -q > $OUT/b.log 2>&1
timeout 120 python tools/microbench.py > $OUT/m.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_kernel -s 3 -c 1 -o $OUT/attn python tools/microbench.py attn > $OUT/ncu.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err

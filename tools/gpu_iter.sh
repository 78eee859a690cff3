# iteration run: kernel tests, bf16 tests, microbench (ping-pong on/off), bench, ncu of relay kernels
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py -q > $OUT/k.log 2>&1
timeout 120 python tools/microbench.py > $OUT/m1.log 2>&1
RK_ATTN_PINGPONG=0 timeout 120 python tools/microbench.py attn > $OUT/m0.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
RK_ATTN_PINGPONG=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench0.json 2> $OUT/bench0.err
for pat in score_kernel select_relay_kernel realign_graft_kernel; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$pat -c 1 -o $OUT/full_$pat python bench.py --steps 1 --warmup 0 --no-cpu --lean > $OUT/ncu_$pat.log 2>&1
done

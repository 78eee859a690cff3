cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02k; mkdir -p $OUT
B="python bench.py --steps 10 --warmup 3 --no-cpu --exact-leg off"
RK_GEMM_LOG=1 timeout 300 $B > $OUT/bench_fix1.json 2> $OUT/bench_fix1.err
RK_GEMM_FIXUP=0 timeout 300 $B > $OUT/bench_fix0.json 2> $OUT/bench_fix0.err
timeout 300 python tools/attn_trace.py 4032 4032 32 8 64 > $OUT/attn_trace_band.txt 2>&1
NV="--nvtx --nvtx-include relay_step/"
LEAN="python bench.py --steps 1 --warmup 0 --no-cpu --lean"
timeout 900 ncu $NV --set full --import-source on --clock-control none -k regex:gemm_bf16_kernel -s 11 -c 4 -o $OUT/full_gemm_sparse $LEAN > $OUT/ncu_gemm_sparse.log 2>&1
timeout 900 ncu $NV --set full --import-source on --clock-control none -k regex:gemm_bf16_kernel -s 0 -c 3 -o $OUT/full_gemm_m320 $LEAN > $OUT/ncu_gemm_m320.log 2>&1
timeout 600 ncu $NV --set full --import-source on --clock-control none -k regex:attn_kernel -s 3 -c 1 -o $OUT/full_attn_sparse $LEAN > $OUT/ncu_attn.log 2>&1

cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02i; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_kernels.py tests/test_gpu_bf16.py -x -q > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
for sw in 2 3; do RK_ATTN_SPLITWAVES=$sw timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_sw$sw.json 2> $OUT/bench_sw$sw.err; done
for g in 1 0; do RK_DECODE_GRAPH=$g timeout 600 python tools/capture_bench.py c2 256 > $OUT/capture_c2_g$g.json 2>&1; done
timeout 600 python tools/capture_bench.py c3 128 > $OUT/capture_c3_g1.json 2>&1
NV="--nvtx --nvtx-include relay_step/"
LEAN="python bench.py --steps 1 --warmup 0 --no-cpu --lean"
for spec in "realign_graft:0"; do
  pat=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu $NV --set full --import-source on --clock-control none -k regex:$pat -s $skip -c 1 -o $OUT/full_${pat}_$skip $LEAN > $OUT/ncu_${pat}_$skip.log 2>&1
done

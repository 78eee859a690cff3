cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_kernels.py -x -q > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
NV="--nvtx --nvtx-include relay_step/"
LEAN="python bench.py --steps 1 --warmup 0 --no-cpu --lean"
for spec in "realign_graft:0" "score_dh_kernel:0"; do
  pat=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu $NV --set full --import-source on --clock-control none -k regex:$pat -s $skip -c 1 -o $OUT/full_${pat}_$skip $LEAN > $OUT/ncu_${pat}_$skip.log 2>&1
done
timeout 900 ncu $NV --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $LEAN > $OUT/launches_bench.log 2>&1

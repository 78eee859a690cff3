cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02u; mkdir -p $OUT
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
NV="--nvtx --nvtx-include relay_step/"
LEAN="python bench.py --steps 1 --warmup 0 --no-cpu --lean"
timeout 600 ncu $NV --set full --import-source on --clock-control none -k regex:score_dh_kernel -s 0 -c 1 -o $OUT/full_score $LEAN > $OUT/ncu_score.log 2>&1
timeout 600 ncu $NV --set full --import-source on --clock-control none -k regex:select_relay -s 0 -c 1 -o $OUT/full_select $LEAN > $OUT/ncu_select.log 2>&1

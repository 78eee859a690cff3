# r02bk-r02bn: host-side timing of agent_prefill (RK_HOST_TIMING) around the result staging change
cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02bn; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for i in 1 2; do RK_HOST_TIMING=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_$i.json 2> $OUT/bench_$i.err; done

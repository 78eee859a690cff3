# full GPU check: all gpu tests, smoke, bench, relay-kernel ncu captures
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "exit $?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
for pat in score_dh_kernel select_relay_kernel realign_graft_dh_kernel; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$pat -c 1 -o $OUT/full_$pat python bench.py --steps 1 --warmup 0 --no-cpu --lean > $OUT/ncu_$pat.log 2>&1
done

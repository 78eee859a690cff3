#!/bin/bash
OUT=gpurun_out/sweep2; mkdir -p $OUT
timeout 2400 python tools/sweep.py > $OUT/sweep_c5.jsonl 2> $OUT/sweep.err
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err
echo done

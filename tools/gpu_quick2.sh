#!/bin/bash
OUT=gpurun_out/q2; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py -q -x > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/b.json 2> $OUT/b.err
python -c "import json; d=json.load(open('$OUT/b.json')); print('bench', d['ms_per_step'], d['roofline']['frac'], d['kernels']['gemm_bf16_tcgen05']['ms'], d['e2e']['ttft_ms'])"
timeout 600 ncu --nvtx --nvtx-include relay_step/ --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu --lean > $OUT/l.log 2>&1
python tools/ncu_summary.py $OUT | head -40

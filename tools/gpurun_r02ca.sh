cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02ca; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k attention > $OUT/pytest_attn.log 2>&1; echo "exit $?" >> $OUT/pytest_attn.log
for c in 1 0 1 0; do echo "COOP=$c" >> $OUT/rows.txt; RK_ATTN_COOP=$c timeout 300 python tools/microbench.py rows >> $OUT/rows.txt 2>&1; done
RK_ATTN_COOP=1 python tools/attn_cta_spans.py pre_suf suffix64 > $OUT/spans.txt 2>&1
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_on_$i.json 2> $OUT/bench_on_$i.err
  RK_ATTN_COOP=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_off_$i.json 2> $OUT/bench_off_$i.err
done

cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02bg; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
python tools/attn_cta_spans.py > $OUT/spans.txt 2>&1
python tools/microbench.py rows > $OUT/rows.txt 2>&1
python tools/microbench.py attn > $OUT/attn.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_$i.json 2> $OUT/bench_$i.err; done

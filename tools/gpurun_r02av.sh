cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02av; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for p in 0x88 0x00 0xAA; do echo "== POLY $p" >> $OUT/mb.txt; RK_ATTN_POLY=$p timeout 120 python tools/microbench.py rows >> $OUT/mb.txt 2>&1; RK_ATTN_POLY=$p timeout 200 python tools/microbench.py attn >> $OUT/mb.txt 2>&1; done

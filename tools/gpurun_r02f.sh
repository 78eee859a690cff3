cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02f; mkdir -p $OUT
MB="import sys; sys.path.insert(0,'.'); from tools.microbench import gemm; from paper_2603_13289_b200.engine import Engine; e=Engine(0)"
RK_GEMM_SWAP=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_swap -s 2 -c 1 -o $OUT/swap_gu320 \
  python -c "$MB; gemm(e,320,16384,2048,2,iters=4)" > $OUT/ncu_swap_gu320.log 2>&1
RK_GEMM_SWAP=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_swap -s 2 -c 1 -o $OUT/swap_qkv320 \
  python -c "$MB; gemm(e,320,3072,2048,3,iters=4)" > $OUT/ncu_swap_qkv320.log 2>&1
RK_GEMM_SWAP=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o $OUT/bf16_gu320 \
  python -c "$MB; gemm(e,320,16384,2048,2,iters=4)" > $OUT/ncu_bf16_gu320.log 2>&1
RK_GEMM_SWAP=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o $OUT/bf16_wo1360 \
  python -c "$MB; gemm(e,1360,2048,2048,1,iters=4)" > $OUT/ncu_bf16_wo1360.log 2>&1

cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02bb; mkdir -p $OUT
python - > $OUT/m320.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, ".")
from tools.microbench import gemm, Engine
e = Engine(0)
for (M, N, K, epi) in [(320, 3072, 2048, 0), (320, 2048, 2048, 1), (320, 2048, 8192, 1), (320, 2048, 2048, 3), (320, 3072, 2048, 3)]:
    for it in (1, 50):
        ms, tf = gemm(e, M, N, K, epi, it)
        print(f"M={M} N={N} K={K} epi={epi} iters={it}: {ms*1e3:.2f} us {tf:.0f} TF/s", flush=True)
PY
for s in "320 3072 2048 0" "320 2048 2048 1" "320 2048 8192 1"; do
  RK_GEMM_LOG=1 python tools/gemm_trace.py $s > "$OUT/trace_${s// /_}.txt" 2>&1
done

cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02bc; mkdir -p $OUT
run() { python - <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, ctypes as C
from tools.microbench import Engine, attn_rows, c2_layout, lib, P, _check
e = Engine(0)
ms, tf = attn_rows(e, "pre_suf", iters=50); print(f"pre_suf {ms*1e3:.1f} us", end="  ")
ms, tf = attn_rows(e, "sparse", iters=50); print(f"sparse {ms*1e3:.1f} us", end="  ")
# suffix only / prefix only
T = 4032
for name, pos in (("suffix64", np.arange(T - 64, T)), ("prefix256", np.arange(256))):
    pos = pos.astype(np.int32); M = len(pos)
    ms = C.c_float()
    _check(lib().rk_debug_bench_attention_rows(P(e.ptr), pos.ctypes.data_as(C.POINTER(C.c_int32)), M, M, M, M, T, 32, 8, 64, 50, C.byref(ms)))
    print(f"{name} {ms.value*1e3:.1f} us", end="  ")
print()
PY
}
for mp in 2 4 8 16 32; do for sd in 1 2 4; do echo -n "MINPART=$mp SPLITDIV=$sd: " >> $OUT/sweep.txt; RK_ATTN_MINPART=$mp RK_ATTN_SPLITDIV=$sd run >> $OUT/sweep.txt 2>&1; done; done

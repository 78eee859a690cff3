import sys, numpy as np
sys.path.insert(0, '.')
from paper_2603_13289_b200.engine import Engine
from paper_2603_13289_b200.abi import ModelSpec
from tests.scenarios import pattern_tokens
e = Engine(0)
def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30))
for name, spec in [("d256_h4_kv2_dh64", ModelSpec.make(4, 256, 4, 2, 64, 512, 256, 10000.0, 2048)),
                   ("d256_h4_kv4_dh64", ModelSpec.make(4, 256, 4, 4, 64, 512, 256, 10000.0, 2048)),
                   ("d512_h8_kv8_dh64", ModelSpec.make(2, 512, 8, 8, 64, 1024, 256, 10000.0, 2048)),
                   ("d512_h4_kv4_dh128", ModelSpec.make(3, 512, 4, 4, 128, 1024, 320, 500000.0, 2048)),
                   ("d256_h2_kv2_dh128", ModelSpec.make(2, 256, 2, 2, 128, 512, 256, 10000.0, 2048))]:
    for n in (57, 130):
        out = {}
        for prec in ("fp32", "bf16"):
            w = e.weights(spec, 99, prec)
            ctx = w.context()
            lg = ctx.prefill(pattern_tokens(n, spec.vocab_size, 2))
            out[prec] = (lg, ctx.all())
        (le, (Ke, Ve)), (lb, (Kb, Vb)) = out["fp32"], out["bf16"]
        per_layer = [(round(rel(Kb[l], Ke[l]), 4), round(rel(Vb[l], Ve[l]), 4)) for l in range(spec.num_layers)]
        nanrows = [int(np.isnan(Kb[l]).any(1).sum()) for l in range(spec.num_layers)]
        print(name, n, "logits", round(rel(lb, le), 4), "K/V per layer", per_layer, "nan rows", nanrows, flush=True)

"""Generate the golden vectors in tests/golden/ from the REFERENCE itself
(oracle/_ref/librelaykv_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run in the build container:  python tests/golden/make_golden.py

Each fixture is a small .npz: the scenario inputs (spec, seeds, tokens), the
reference's decode-time RelayCache (small specs only; hashed otherwise) and the
outputs of relay_prefill / the agent TTFT sequence: selection, tags, s_dev,
s_key_dev, depth, marks, stats, logits (bit patterns), and SHA-256 digests of
the merged KV context and segment hidden states.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle  # noqa: E402
from tests.golden.cases import CASES  # noqa: E402


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run_case(orc, case):
    spec, w = case["spec"](), None
    w = orc.weights(spec, case["seed"], checked=case.get("checked", False))
    caches = [orc.scenario(w, old, n, snap) for (old, n, snap) in case["upstream"]]
    out = {"cache_digests": [digest(c.segment_tokens, c.k_pre, c.v, c.hidden_snapshot, c.influence)
                             for c in caches]}
    if case["kind"] == "relay_prefill":
        o, ctx = orc.relay_prefill(w, case["prefix"], caches[0], case["profile"], case["opts"])
        K, V = orc.ctx_all(ctx)
        out.update({
            "selection": o["selection"], "tags": o["tags"], "s_dev": o["s_dev"], "s_key_dev": o["s_key_dev"],
            "depth": o["depth"], "origin": o["origin"], "logits": o["logits"],
            "hidden_digest": digest(o["hidden"]), "ctx_digest": digest(K, V),
            "stats": {k: v for k, v in o["stats"].items() if k != "wall"},
        })
    else:
        logits, tok, ctx = orc.agent_prefill(w, case["prefix"], caches, case["suffix"], case["profile"], case["opts"])
        K, V = orc.ctx_all(ctx)
        out.update({"logits": logits, "first_token": tok, "ctx_digest": digest(K, V),
                    "marks": [s[2] for s in orc.ctx_segments(ctx)]})
    return caches, out


def main():
    orc = Oracle("reference")
    for name, case in CASES.items():
        caches, out = run_case(orc, case)
        arrays = {}
        meta = {"name": name, "generator": "oracle/_ref (reference library built from /root/reference/proj/src)"}
        for k, v in out.items():
            if isinstance(v, np.ndarray):
                arrays[k] = v
            elif k == "marks":
                for i, m in enumerate(v):
                    arrays[f"marks_{i}"] = m
            else:
                meta[k] = v
        if case.get("store_cache"):
            c = caches[0]
            arrays.update({"cache_k_pre": c.k_pre, "cache_v": c.v, "cache_hidden": c.hidden_snapshot,
                           "cache_influence": c.influence, "cache_tokens": c.segment_tokens})
        arrays["meta"] = np.frombuffer(json.dumps(meta, default=float).encode(), dtype=np.uint8)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
        print(name, {k: (v.shape if hasattr(v, 'shape') else v) for k, v in arrays.items() if k != "meta"})


if __name__ == "__main__":
    main()

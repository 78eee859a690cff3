"""Golden RKRC relay-cache files written by the REFERENCE itself
(save_relay_cache, relay_cache.cpp:238-245, via oracle/_ref). Run in the
build container:  python tests/golden/make_rkrc.py

Each <name>.rkrc is the decode-time capture of one upstream scenario of
cases.py (same spec, weight seed, old prefix, segment length, snapshot layer),
so the engine can re-capture the same cache on the GPU and must save a file
byte-identical to it. <name>.rkrc.json records the scenario.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle  # noqa: E402
from tests.golden.cases import CASES  # noqa: E402

# (file name, case, upstream index)
FILES = [("cache_diag_L8_d32", "relay_diag_L8_d32", 0), ("cache_gqa_L6_d64", "agent_gqa_two_segments", 0)]


def main():
    orc = Oracle("reference")
    for name, case_name, i in FILES:
        case = CASES[case_name]
        spec = case["spec"]()
        w = orc.weights(spec, case["seed"], checked=case.get("checked", False))
        old, n, snap = case["upstream"][i]
        host = orc.scenario(w, old, n, snap)
        path = os.path.join(HERE, f"{name}.rkrc")
        orc.save_cache(host, path)
        meta = {"case": case_name, "upstream": i, "seed": case["seed"], "checked": case.get("checked", False),
                "old_prefix": [int(t) for t in old], "segment_len": n, "snapshot_layer": snap,
                "generator": "oracle/_ref save_relay_cache"}
        with open(path + ".json", "w") as f:
            json.dump(meta, f, indent=1)
        print(name, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

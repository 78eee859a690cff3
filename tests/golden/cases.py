"""Golden-vector scenarios (inputs only; outputs come from the reference via
make_golden.py). Mirrors the reference's own test scenarios
(test_engine.cpp:101-324) plus BASELINE config 1."""
from paper_2603_13289_b200.abi import LayerProfile, RelayOptions
from tests.scenarios import c1_spec, pattern_tokens, spec_of, synthetic_tokens, triple

CASES = {
    # test_engine.cpp:298-324 "selection diagnostics are exposed and consistent"
    "relay_diag_L8_d32": dict(kind="relay_prefill", spec=lambda: spec_of(8, 32, 4), seed=108,
                              upstream=[(pattern_tokens(14, 64, 0), 20, 1)], prefix=pattern_tokens(10, 64, 8),
                              profile=triple(1, 3, 6), opts=RelayOptions.make(suffix_k=4), store_cache=True,
                              checked=True),
    # test_engine.cpp:139-178 accounting: (1,3,18) on 32 layers, N=100
    "relay_accounting_L32": dict(kind="relay_prefill", spec=lambda: spec_of(32, 16, 2), seed=103,
                                 upstream=[(pattern_tokens(8, 64, 0), 100, 1)], prefix=pattern_tokens(12, 64, 3),
                                 profile=triple(1, 3, 18),
                                 opts=RelayOptions.make(tau_dev=1e9, tau_inf=1e9, suffix_k=10), checked=True),
    # test_engine.cpp:180-208 blend baseline
    "blend_alpha02_L8": dict(kind="relay_prefill", spec=lambda: spec_of(8, 32, 4), seed=104,
                             upstream=[(pattern_tokens(10, 64, 0), 12, 0)], prefix=pattern_tokens(7, 64, 9),
                             profile=LayerProfile(), opts=RelayOptions.make(mode="blend", blend_alpha=0.25),
                             checked=True),
    # BASELINE config 1: 2 layers, d=256, 4 heads, 512-token segment (unchecked init mirror)
    "c1_relay_L2_d256_N512": dict(kind="relay_prefill", spec=c1_spec, seed=1234,
                                  upstream=[(synthetic_tokens(1234, 1, 64, 256), 512, 0)],
                                  prefix=synthetic_tokens(1234, 2, 48, 256), profile=triple(0, 0, 1),
                                  opts=RelayOptions.make()),
    # workflow.cpp:316-369: prefix + 2 relayed segments + suffix, GQA
    "agent_gqa_two_segments": dict(kind="agent", spec=lambda: spec_of(6, 64, 4, kv_heads=2), seed=77,
                                   upstream=[(pattern_tokens(9, 64, 1), 16, 1), (pattern_tokens(7, 64, 2), 11, 1)],
                                   prefix=pattern_tokens(5, 64, 3), suffix=pattern_tokens(4, 64, 4),
                                   profile=triple(1, 2, 4), opts=RelayOptions.make(suffix_k=3), checked=True),
}


# ---- measured-width cases (tests/golden/make_golden_wide.py -> tests/golden/wide/) ----
# Full model width of BASELINE config 2 (Llama-3.2-1B shape) and config 3
# (Llama-3-8B shape) with a chain the reference finishes in minutes. Same
# seed, profile and thresholds as bench.py's workloads.
def c2_spec():
    from paper_2603_13289_b200.abi import ModelSpec
    return ModelSpec.make(16, 2048, 32, 8, 64, 8192, 128256, 500000.0, 8192)


def c3_spec():
    from paper_2603_13289_b200.abi import ModelSpec
    return ModelSpec.make(32, 4096, 32, 8, 128, 14336, 128256, 500000.0, 16384)


_V = 128256
WIDE_CASES = {
    # c2 width: prefix 32 + 2 relayed decode-time segments x 128 + suffix 8, profile (1,2,9)
    "c2w_chain_2x128": dict(spec=c2_spec, spec_id="c2", seed=1234,
                            upstream=[(synthetic_tokens(1234, 0, 32, _V), 128, 1),
                                      (synthetic_tokens(1234, 3, 32, _V), 128, 1)],
                            prefix=synthetic_tokens(1234, 6, 32, _V), suffix=synthetic_tokens(1234, 7, 8, _V),
                            profile=triple(1, 2, 9), opts=RelayOptions.make(tau_dev=1.5, tau_inf=1.45, suffix_k=10),
                            describe="c2 width (L16 d2048 H32/8 dh64 ff8192 V128256), prefix 32 + 2x128 + suffix 8, "
                                     "profile (1,2,9)"),
    # c3 width: prefix 16 + 1 relayed segment x 64 + suffix 4, profile (1,3,18)
    "c3w_chain_1x64": dict(spec=c3_spec, spec_id="c3", seed=1234,
                           upstream=[(synthetic_tokens(1234, 0, 16, _V), 64, 1)],
                           prefix=synthetic_tokens(1234, 6, 16, _V), suffix=synthetic_tokens(1234, 7, 4, _V),
                           profile=triple(1, 3, 18), opts=RelayOptions.make(tau_dev=1.5, tau_inf=1.45, suffix_k=10),
                           describe="c3 width (L32 d4096 H32/8 dh128 ff14336 V128256), prefix 16 + 1x64 + suffix 4, "
                                    "profile (1,3,18)"),
}

"""Shared scenario builders, mirroring the reference tests' helpers
(test_engine.cpp:14-33, 43-62, 64-76)."""
import numpy as np

from paper_2603_13289_b200.abi import LayerProfile, ModelSpec, RelayOptions


def spec_of(layers, d_model, heads, kv_heads=None, vocab=64, max_positions=4096, d_ff=None,
            theta=10000.0):
    """spec_of (test_engine.cpp:14-25): d_head = d/heads, d_ff = 2d."""
    return ModelSpec.make(layers, d_model, heads, kv_heads or heads, d_model // heads,
                          d_ff or 2 * d_model, vocab, theta, max_positions)


def pattern_tokens(n, vocab, salt):
    """pattern_tokens (test_engine.cpp:27-33)."""
    return np.array([(i * 13 + salt * 7 + 1) % vocab for i in range(n)], np.int32)


def triple(a, b, c):
    return LayerProfile(a, b, c)


def c1_spec():
    """BASELINE config 1: 2 layers, d=256, 4 heads."""
    return ModelSpec.make(2, 256, 4, 4, 64, 512, 256, 10000.0, 1024)


def synthetic_tokens(seed, salt, count, vocab):
    """synthetic_tokens (metrics.cpp:255-263)."""
    mask = (1 << 64) - 1
    state = (seed ^ ((salt * 0x9e3779b97f4a7c15 + 0x1234567) & mask)) & mask
    out = np.empty(count, np.int32)
    for i in range(count):
        state = (state + 0x9e3779b97f4a7c15) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & mask
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & mask
        z = z ^ (z >> 31)
        out[i] = z % vocab
    return out


# Parity scenarios: (name, spec, weight seed, old prefix, segment len, snapshot,
#                    new prefix, profile, options)
def parity_scenarios():
    out = []
    s8 = spec_of(8, 32, 4)
    out.append(("relay_1_3_6", s8, 108, pattern_tokens(14, 64, 0), 20, 1, pattern_tokens(10, 64, 8),
                triple(1, 3, 6), RelayOptions.make(suffix_k=4)))
    out.append(("relay_default", s8, 106, pattern_tokens(10, 64, 0), 8, 1, pattern_tokens(6, 64, 4),
                triple(1, 2, 5), RelayOptions.make()))
    out.append(("degenerate_full", s8, 101, pattern_tokens(12, 64, 0), 10, 0, pattern_tokens(9, 64, 5),
                triple(0, 0, 7), RelayOptions.make(suffix_k=10)))
    out.append(("full_mode", s8, 101, pattern_tokens(12, 64, 0), 10, 0, pattern_tokens(9, 64, 5),
                triple(0, 0, 7), RelayOptions.make(mode="full")))
    out.append(("zero_mode", s8, 102, pattern_tokens(10, 64, 0), 8, 2, pattern_tokens(10, 64, 0),
                LayerProfile(), RelayOptions.make(mode="zero")))
    out.append(("blend_alpha_1", s8, 104, pattern_tokens(10, 64, 0), 12, 0, pattern_tokens(7, 64, 9),
                LayerProfile(), RelayOptions.make(mode="blend", blend_alpha=1.0)))
    out.append(("blend_alpha_03", s8, 104, pattern_tokens(10, 64, 0), 12, 0, pattern_tokens(7, 64, 9),
                LayerProfile(), RelayOptions.make(mode="blend", blend_alpha=0.3)))
    gqa = ModelSpec.make(6, 64, 4, 2, 16, 128, 64, 10000.0, 1024)
    out.append(("gqa_relay", gqa, 7, pattern_tokens(16, 64, 2), 24, 1, pattern_tokens(11, 64, 3),
                triple(1, 2, 4), RelayOptions.make(suffix_k=3)))
    out.append(("rectify_above_end", gqa, 9, pattern_tokens(9, 64, 1), 16, 2, pattern_tokens(13, 64, 6),
                triple(2, 3, 3), RelayOptions.make(suffix_k=2, rectify_above_end=True)))
    return out

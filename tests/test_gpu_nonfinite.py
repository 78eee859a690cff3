"""ensure_finite (tensor.cpp:58-64): the reference throws runtime_error
("<what>: non-finite value") after any matmul that produced inf/NaN. The
engine raises NonFiniteError (RK_ERR_NONFINITE) from the device flag, in
both precisions: the fp32-exact SIMT GEMM, and the bf16 tcgen05 GEMM
epilogues (QKV / residual / SiLU / split-K reduce / GEMV) and attention."""
import numpy as np
import pytest

from paper_2603_13289_b200.abi import LayerProfile, ModelSpec, NonFiniteError, RelayOptions
from tests.scenarios import pattern_tokens

pytestmark = pytest.mark.gpu

SPEC = ModelSpec.make(4, 256, 4, 2, 64, 512, 256, 10000.0, 2048)
# tensor_table order (weights_io.cpp:21-38): embedding, then per layer
# attn_norm, w_q, w_k, w_v, w_o, mlp_norm, w_gate, w_up, w_down; final norm, head
W_Q, W_K, W_GATE, HEAD = 1 + 1, 1 + 2, 1 + 6, 1 + 9 * 4 + 1


def tensors(oracle, seed=31):
    ow = oracle.weights(SPEC, seed)
    n = 3 + 9 * SPEC.num_layers
    return [oracle.weights_tensor(ow, i) for i in range(n)], ow


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("where", ["w_q_inf", "w_gate_nan", "head_inf", "scores_overflow"])
def test_nonfinite_raises(engine, oracle, precision, where):
    ts, ow = tensors(oracle)
    ts = [t.copy() for t in ts]
    if where == "w_q_inf":
        ts[W_Q][5] = np.inf               # QKV GEMM of layer 0
    elif where == "w_gate_nan":
        ts[W_GATE][17] = np.nan           # gate/up GEMM (SiLU epilogue)
    elif where == "head_inf":
        ts[HEAD][3] = -np.inf             # logits head (GEMV)
    else:                                 # finite projections whose q.k overflows fp32: attention
        ts[W_Q] *= 1e19
        ts[W_K] *= 1e19
    w = engine.weights_from_tensors(SPEC, ts, precision)
    prompt = pattern_tokens(40, SPEC.vocab_size, 1)
    with pytest.raises(NonFiniteError):
        w.context().prefill(prompt)
    # the flag is per call: the same engine keeps working on finite weights
    good = engine.weights_from_tensors(SPEC, tensors(oracle)[0], precision)
    assert np.all(np.isfinite(good.context().prefill(prompt)))


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_nonfinite_in_relay_path(engine, oracle, precision):
    """A non-finite value produced inside the relay step (the band recompute)
    fails the relay call like the reference's relay_prefill would."""
    ts, ow = tensors(oracle)
    cache = oracle.scenario(ow, pattern_tokens(30, 256, 1), 200, 1)
    bad = [t.copy() for t in ts]
    bad[1 + 9 * 1 + 6][11] = np.inf  # layer 1 (the band) gate weights
    w = engine.weights_from_tensors(SPEC, bad, precision)
    with pytest.raises(NonFiniteError):
        w.context().relay_prefill(pattern_tokens(20, 256, 2), w.upload_cache(cache), LayerProfile(1, 1, 2),
                                  RelayOptions.make(suffix_k=4))

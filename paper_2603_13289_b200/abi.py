"""ctypes mirror of include/relaykv_b200.h (the C ABI of the engine).

Struct layouts here must match the header field for field; tests/test_abi.py
checks sizes against the compiled library.
"""
import ctypes as C

RK_OK = 0
RK_ERR_INVALID_ARGUMENT = 1
RK_ERR_SCHEMA = 2
RK_ERR_LOGIC = 3
RK_ERR_NONFINITE = 4
RK_ERR_RUNTIME = 5
RK_ERR_IO = 6

RK_FP32_EXACT = 0
RK_BF16 = 1
RK_FP32_TC = 2

RK_MODE_FULL = 0
RK_MODE_ZERO = 1
RK_MODE_RELAY = 2
RK_MODE_BLEND = 3

RK_SEL_DEVIATION = 1
RK_SEL_INFLUENCE_SCORE = 2
RK_SEL_INFLUENCE_SUFFIX = 4
RK_SEL_BLEND_TOPK = 8

MODES = {"full": RK_MODE_FULL, "zero": RK_MODE_ZERO, "relay": RK_MODE_RELAY, "blend": RK_MODE_BLEND}


class ModelSpec(C.Structure):
    """rk_model_spec == relaykv::ModelSpec (model.hpp:21-38)."""
    _fields_ = [
        ("num_layers", C.c_uint64),
        ("d_model", C.c_uint64),
        ("num_heads", C.c_uint64),
        ("num_kv_heads", C.c_uint64),
        ("d_head", C.c_uint64),
        ("d_ff", C.c_uint64),
        ("vocab_size", C.c_uint64),
        ("theta_base", C.c_float),
        ("max_positions", C.c_uint64),
        ("norm_eps", C.c_float),
    ]

    @classmethod
    def make(cls, num_layers, d_model, num_heads, num_kv_heads=None, d_head=None, d_ff=None,
             vocab_size=64, theta_base=10000.0, max_positions=4096, norm_eps=1e-5):
        num_kv_heads = num_kv_heads or num_heads
        d_head = d_head or d_model // num_heads
        d_ff = d_ff or 2 * d_model
        return cls(num_layers, d_model, num_heads, num_kv_heads, d_head, d_ff, vocab_size,
                   theta_base, max_positions, norm_eps)

    @property
    def kv_dim(self):
        return self.num_kv_heads * self.d_head

    @property
    def q_dim(self):
        return self.num_heads * self.d_head

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class LayerProfile(C.Structure):
    """rk_layer_profile == LayerProfile window (profiler.hpp:30-43)."""
    _fields_ = [("l_start", C.c_uint64), ("l_det", C.c_uint64), ("l_end", C.c_uint64)]


class RelayOptions(C.Structure):
    """rk_relay_options == RelayOptions + SelectionThresholds (relay_engine.hpp:119-126)."""
    _fields_ = [
        ("mode", C.c_int32),
        ("tau_dev", C.c_double),
        ("tau_inf", C.c_double),
        ("suffix_k", C.c_uint64),
        ("blend_alpha", C.c_double),
        ("rectify_above_end", C.c_int32),
    ]

    @classmethod
    def make(cls, mode="relay", tau_dev=1.5, tau_inf=1.45, suffix_k=10, blend_alpha=0.2,
             rectify_above_end=False):
        m = MODES[mode] if isinstance(mode, str) else int(mode)
        return cls(m, tau_dev, tau_inf, suffix_k, blend_alpha, int(rectify_above_end))


class RelayCacheView(C.Structure):
    """rk_relay_cache_view == RelayCache (relay_cache.hpp:23-46)."""
    _fields_ = [
        ("num_layers", C.c_uint64),
        ("num_kv_heads", C.c_uint64),
        ("d_head", C.c_uint64),
        ("d_model", C.c_uint64),
        ("theta_base", C.c_float),
        ("max_positions", C.c_uint64),
        ("segment_len", C.c_uint64),
        ("segment_tokens", C.POINTER(C.c_int32)),
        ("source_base_position", C.c_uint64),
        ("snapshot_layer", C.c_uint64),
        ("decode_steps_observed", C.c_uint64),
        ("k_pre", C.POINTER(C.POINTER(C.c_float))),
        ("v", C.POINTER(C.POINTER(C.c_float))),
        ("hidden_snapshot", C.POINTER(C.c_float)),
        ("influence", C.POINTER(C.c_float)),
    ]


class PhaseTimings(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("fresh_ms", "realign_ms", "recompute_ms", "selection_ms", "rectify_ms", "total_ms")]


class ReuseStats(C.Structure):
    """rk_reuse_stats == ReuseStats (relay_engine.hpp:53-71)."""
    _fields_ = [
        ("total_entries", C.c_uint64),
        ("recomputed_entries", C.c_uint64),
        ("reuse_rate", C.c_double),
        ("selected_count", C.c_uint64),
        ("selected_deviation", C.c_uint64),
        ("selected_influence_score", C.c_uint64),
        ("selected_influence_suffix", C.c_uint64),
        ("selected_blend", C.c_uint64),
        ("flops_cost", C.c_double),
        ("flops_selection", C.c_double),
        ("flops_realign", C.c_double),
        ("flops_full_equiv", C.c_double),
        ("wall", PhaseTimings),
    ]


class RelayOutput(C.Structure):
    """rk_relay_output == RelayOutput (relay_engine.hpp:128-137) + SegmentMarks."""
    _fields_ = [
        ("selection_indices", C.POINTER(C.c_uint64)),
        ("selection_tags", C.POINTER(C.c_uint32)),
        ("s_dev", C.POINTER(C.c_double)),
        ("s_key_dev", C.POINTER(C.c_double)),
        ("segment_hidden", C.POINTER(C.c_float)),
        ("hidden_depth", C.POINTER(C.c_uint64)),
        ("origin", C.POINTER(C.c_uint8)),
        ("segment_base", C.c_uint64),
        ("segment_len", C.c_uint64),
        ("selection_count", C.c_uint64),
        ("s_dev_len", C.c_uint64),
        ("dev_threshold", C.c_double),
        ("min_dev_margin", C.c_double),
        ("stats", ReuseStats),
    ]


class ProfilerParams(C.Structure):
    """rk_profiler_params == ProfilerParams (profiler.hpp:19-28)."""
    _fields_ = [
        ("tau_start", C.c_double),
        ("tail_layers", C.c_uint64),
        ("stability_lambda", C.c_double),
        ("consecutive", C.c_uint64),
        ("min_rise", C.c_uint64),
        ("first_negative_alpha", C.c_int32),
    ]

    @classmethod
    def make(cls, tau_start=0.99, tail_layers=5, stability_lambda=2.0, consecutive=2, min_rise=3,
             first_negative_alpha=False):
        return cls(tau_start, tail_layers, stability_lambda, consecutive, min_rise, int(first_negative_alpha))


class TwoStageConfig(C.Structure):
    """rk_two_stage_config == TwoStageConfig (metrics.hpp:93-107)."""
    _fields_ = [
        ("seed", C.c_uint64),
        ("instances", C.c_uint64),
        ("stage1_prefix_min", C.c_uint64),
        ("stage1_prefix_max", C.c_uint64),
        ("stage2_prefix_min", C.c_uint64),
        ("stage2_prefix_max", C.c_uint64),
        ("segment_len", C.c_uint64),
        ("stage2_suffix_len", C.c_uint64),
        ("sweep_instances", C.c_uint64),
        ("identical_prefix", C.c_int32),
        ("snapshot_layer", C.c_uint64),
    ]

    @classmethod
    def make(cls, seed=1, instances=8, stage1_prefix=(32, 64), stage2_prefix=(24, 72), segment_len=48,
             stage2_suffix_len=16, sweep_instances=2, identical_prefix=False, snapshot_layer=0):
        return cls(seed, instances, stage1_prefix[0], stage1_prefix[1], stage2_prefix[0], stage2_prefix[1],
                   segment_len, stage2_suffix_len, sweep_instances, int(identical_prefix), snapshot_layer)


class ProfileResult(C.Structure):
    """rk_profile_result: the LayerProfile window + fallback warnings (profiler.cpp:123-155)."""
    _fields_ = [("l_start", C.c_uint64), ("l_det", C.c_uint64), ("l_end", C.c_uint64),
                ("end_fallback", C.c_int32), ("det_fallback", C.c_int32)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


def stats_dict(st):
    d = {f: getattr(st, f) for f, _ in ReuseStats._fields_ if f != "wall"}
    d["wall"] = {f: getattr(st.wall, f) for f, _ in PhaseTimings._fields_}
    return d


class StatusError(RuntimeError):
    """Raised for a non-zero rk_status; .code is the rk_status."""

    def __init__(self, code, msg):
        super().__init__(f"[rk_status {code}] {msg}")
        self.code = code


def exception_for(code, msg):
    """Map an rk_status to the exception type the reference throws (errors.hpp,
    SURVEY.md 8(b)): invalid_argument -> ValueError, SchemaError -> SchemaError,
    logic_error -> LogicError, IoError -> IoError (an OSError),
    non-finite/runtime -> RuntimeError subclasses."""
    cls = {RK_ERR_INVALID_ARGUMENT: InvalidArgument, RK_ERR_SCHEMA: SchemaError,
           RK_ERR_LOGIC: LogicError, RK_ERR_NONFINITE: NonFiniteError, RK_ERR_IO: IoError}.get(code, StatusError)
    return cls(code, msg)


class InvalidArgument(StatusError, ValueError):
    pass


class SchemaError(StatusError):
    pass


class LogicError(StatusError):
    pass


class NonFiniteError(StatusError):
    pass


class IoError(StatusError, OSError):
    """relaykv::IoError (errors.hpp:12): a file could not be opened/read/written."""

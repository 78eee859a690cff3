"""Offline layer profiler (profiler.hpp / metrics.hpp of the reference):
calibrates the LayerProfile window (l_start, l_det, l_end) a relay uses.

  profile_model(weights, calib, params)     profiler.cpp:157-175, captures,
                                            prefills and token deviations on
                                            the device (rk_profile_model)
  token_deviation(reuse, full)              metrics.cpp:118-159 on the device
  make_layer_curve / average_curves /
  profile_from_curve                        host scans (metrics.cpp:162-238,
                                            profiler.cpp:49-155)

In RK_FP32_EXACT every number is bit-identical to the reference.
"""
import ctypes as C

import numpy as np

from .abi import ProfileResult, ProfilerParams, TwoStageConfig
from .engine import P, U64, _check, lib

F64P = C.POINTER(C.c_double)
U8P = C.POINTER(C.c_uint8)

__all__ = ["ProfilerParams", "TwoStageConfig", "ProfileResult", "profile_model", "token_deviation",
           "make_layer_curve", "average_curves", "profile_from_curve"]


def _d(a):
    return a.ctypes.data_as(F64P)


def token_deviation(reuse, full):
    """DeviationMatrix of two device caches of one segment: dict of four
    [n x L] float64 arrays (value_cos, key_cos, value_norm, key_norm)."""
    L, n = reuse.weights.spec.num_layers, reuse.segment_len
    out = {k: np.empty((n, L), np.float64) for k in ("value_cos", "key_cos", "value_norm", "key_norm")}
    _check(lib().rk_token_deviation(P(reuse.ptr), P(full.ptr), _d(out["value_cos"]), _d(out["key_cos"]),
                                    _d(out["value_norm"]), _d(out["key_norm"])))
    return out


def make_layer_curve(value_cos):
    """s[L], rho[L] (rho[0] NaN), rho_degenerate[L] of a [n x L] deviation matrix."""
    m = np.ascontiguousarray(value_cos, np.float64)
    n, L = m.shape
    s, rho, deg = np.empty(L), np.empty(L), np.empty(L, np.uint8)
    _check(lib().rk_layer_curve(_d(m), U64(n), U64(L), _d(s), _d(rho), deg.ctypes.data_as(U8P)))
    return {"s": s, "rho": rho, "rho_degenerate": deg.astype(bool)}


def average_curves(curves):
    s = np.ascontiguousarray([c["s"] for c in curves], np.float64)
    rho = np.ascontiguousarray([c["rho"] for c in curves], np.float64)
    deg = np.ascontiguousarray([c["rho_degenerate"] for c in curves], np.uint8)
    k, L = s.shape
    so, ro, do = np.empty(L), np.empty(L), np.empty(L, np.uint8)
    _check(lib().rk_average_curves(_d(s), _d(rho), deg.ctypes.data_as(U8P), U64(k), U64(L), _d(so), _d(ro),
                                   do.ctypes.data_as(U8P)))
    return {"s": so, "rho": ro, "rho_degenerate": do.astype(bool)}


def profile_from_curve(curve, params=None):
    params = params or ProfilerParams.make()
    s = np.ascontiguousarray(curve["s"], np.float64)
    rho = np.ascontiguousarray(curve["rho"], np.float64)
    deg = np.ascontiguousarray(curve["rho_degenerate"], np.uint8)
    L = s.shape[0]
    out, crho = ProfileResult(), np.empty(max(L - 1, 1))
    _check(lib().rk_profile_from_curve(_d(s), _d(rho), deg.ctypes.data_as(U8P), U64(L), C.byref(params),
                                       C.byref(out), _d(crho)))
    d = out.as_dict()
    d["curve_s"], d["curve_rho"] = s, crho[:L - 1]
    return d


def profile_model(weights, calib=None, params=None):
    """profile_model on the device: dict with l_start, l_det, l_end, the
    fallback flags and the averaged curves."""
    calib = calib or TwoStageConfig.make()
    params = params or ProfilerParams.make()
    L = weights.spec.num_layers
    out, s, rho = ProfileResult(), np.empty(L), np.empty(max(L - 1, 1))
    _check(lib().rk_profile_model(P(weights.engine.ptr), P(weights.ptr), C.byref(calib), C.byref(params),
                                  C.byref(out), _d(s), _d(rho)))
    d = out.as_dict()
    d["curve_s"], d["curve_rho"] = s, rho[:L - 1]
    return d

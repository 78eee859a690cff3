"""Python host mirror of the relay-prefill C ABI (include/relaykv_b200.h).

Mirrors the reference's API on this path (relay_engine.hpp:142-163,
model.hpp:116-152) with the same argument meaning and error types: every
call goes through librelaykv_b200.so; there is no CPU fallback. A missing
library raises at import of this module.
"""
import ctypes as C
import os
import sys

import numpy as np

from .abi import (LayerProfile, ModelSpec, RelayCacheView, RelayOptions, RelayOutput, RK_BF16,
                  RK_FP32_EXACT, RK_FP32_TC, exception_for, stats_dict)
from .hostcache import HostRelayCache

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librelaykv_b200.so")

P = C.c_void_p
U64 = C.c_uint64
F32P = C.POINTER(C.c_float)
I32P = C.POINTER(C.c_int32)

_lib = None


def lib():
    """Load the engine library (loudly: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2603_13289_b200.build` "
                              "(the relay path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.rk_last_error.restype = C.c_char_p
        L.rk_engine_stream.restype = P
        L.rk_engine_stream.argtypes = [P]
        L.rk_engine_launch_count.restype = U64
        L.rk_engine_launch_count.argtypes = [P]
        for f in ("rk_context_size", "rk_context_num_segments", "rk_cache_segment_len"):
            getattr(L, f).restype = U64
            getattr(L, f).argtypes = [P]
        L.rk_weights_num_tensors.restype = U64
        L.rk_weights_num_tensors.argtypes = [C.POINTER(ModelSpec)]
        for f in ("rk_engine_destroy", "rk_weights_destroy", "rk_cache_destroy", "rk_context_destroy",
                  "rk_cache_file_free"):
            getattr(L, f).restype = None
            getattr(L, f).argtypes = [P]
        L.rk_flops_span_full.restype = C.c_double
        L.rk_flops_span_full.argtypes = [C.POINTER(ModelSpec), U64, U64]
        L.rk_flops_segment_schedule.restype = C.c_double
        L.rk_flops_segment_schedule.argtypes = [C.POINTER(ModelSpec), U64, U64, U64, U64, U64, U64]
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        raise exception_for(st, lib().rk_last_error().decode())


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(I32P)


class _Obj:
    _dtor = None

    def __init__(self, ptr, owner=None):
        self.ptr = ptr
        self._owner = owner  # keep parents alive

    def close(self):
        if getattr(self, "ptr", None):
            getattr(lib(), self._dtor)(P(self.ptr))
            self.ptr = None

    def __del__(self):
        # (at interpreter shutdown the engine may already be gone -- objects
        # kept alive by a traceback must not free into a destroyed engine;
        # the process exit releases the device memory)
        if sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_uint64), ("total_ms", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


class Engine(_Obj):
    """One engine per CUDA device (rk_engine_create)."""
    _dtor = "rk_engine_destroy"

    def __init__(self, device=0):
        out = P()
        _check(lib().rk_engine_create(int(device), C.byref(out)))
        super().__init__(out.value)
        self.device = device

    @property
    def stream(self):
        return lib().rk_engine_stream(P(self.ptr))

    @property
    def launches(self):
        return int(lib().rk_engine_launch_count(P(self.ptr)))

    def synchronize(self):
        _check(lib().rk_engine_synchronize(P(self.ptr)))

    def set_graphs(self, enable):
        _check(lib().rk_engine_set_graphs(P(self.ptr), int(enable)))

    def set_fused(self, enable):
        """Layer-major fused agent schedule (default) vs the sequential order."""
        _check(lib().rk_engine_set_fused(P(self.ptr), int(enable)))

    def profile(self, enable=True):
        """Per-kernel CUDA-event instrumentation of the hot kernels (clears)."""
        _check(lib().rk_engine_profile(P(self.ptr), int(enable)))

    def profile_read(self):
        cap = 64
        while True:  # every aggregated record (a c3 step has a few hundred distinct labels)
            stats = (KernelStat * cap)()
            n = U64()
            _check(lib().rk_engine_profile_read(P(self.ptr), stats, U64(cap), C.byref(n)))
            if n.value <= cap:
                break
            cap = int(n.value)
        return [{"name": stats[i].name.decode(), "launches": int(stats[i].launches),
                 "total_ms": stats[i].total_ms, "flops": stats[i].flops, "bytes": stats[i].bytes}
                for i in range(n.value)]

    # ---- factories ------------------------------------------------------------
    def weights(self, spec, seed, precision="fp32"):
        """init_weights(spec, seed) on the device (model.cpp:81-114)."""
        prec = {"fp32": RK_FP32_EXACT, "bf16": RK_BF16, "fp32tc": RK_FP32_TC}[precision]
        out = P()
        _check(lib().rk_weights_init(P(self.ptr), C.byref(spec), U64(seed), prec, C.byref(out)))
        return Weights(out.value, self, spec, precision)

    def weights_from_tensors(self, spec, tensors, precision="fp32"):
        prec = {"fp32": RK_FP32_EXACT, "bf16": RK_BF16, "fp32tc": RK_FP32_TC}[precision]
        arrs = [np.ascontiguousarray(t, np.float32) for t in tensors]
        ptrs = (F32P * len(arrs))(*[a.ctypes.data_as(F32P) for a in arrs])
        out = P()
        _check(lib().rk_weights_upload(P(self.ptr), C.byref(spec), ptrs, U64(len(arrs)), prec, C.byref(out)))
        return Weights(out.value, self, spec, precision)


class Weights(_Obj):
    _dtor = "rk_weights_destroy"

    def __init__(self, ptr, engine, spec, precision):
        super().__init__(ptr, engine)
        self.engine, self.spec, self.precision = engine, spec, precision

    def num_tensors(self):
        return int(lib().rk_weights_num_tensors(C.byref(self.spec)))

    def tensor(self, idx, numel):
        out = np.empty(numel, np.float32)
        _check(lib().rk_weights_export(P(self.ptr), U64(idx), out.ctypes.data_as(F32P), U64(numel)))
        return out

    def context(self):
        out = P()
        _check(lib().rk_context_create(P(self.engine.ptr), P(self.ptr), C.byref(out)))
        return Context(out.value, self)

    def upload_cache(self, host, asynchronous=False, defer=None):
        """RelayCache host arrays -> device (rk_cache_upload). asynchronous:
        rk_cache_upload_async -- layers stream in on the copy stream while
        later calls run; the host arrays stay referenced by the Cache.
        defer=(lo, hi) (asynchronous only): those layers cross PCIe only when
        a later call reads them (rk_cache_upload_async_defer)."""
        out = P()
        if defer is not None:
            assert asynchronous, "deferred layers need an asynchronous upload"
            _check(lib().rk_cache_upload_async_defer(P(self.engine.ptr), P(self.ptr), C.byref(host.view()),
                                                     U64(defer[0]), U64(defer[1]), C.byref(out)))
        else:
            fn = lib().rk_cache_upload_async if asynchronous else lib().rk_cache_upload
            _check(fn(P(self.engine.ptr), P(self.ptr), C.byref(host.view()), C.byref(out)))
        c = Cache(out.value, self)
        if asynchronous:
            c._host = host
        return c

    def load_cache(self, path, asynchronous=False):
        """load_relay_cache (relay_cache.cpp:247-253) of an RKRC file straight
        onto the device (rk_cache_load). asynchronous: the blob is read into
        pinned memory and streams in layer by layer like upload_cache."""
        out = P()
        _check(lib().rk_cache_load(P(self.engine.ptr), P(self.ptr), os.fsencode(path), int(asynchronous),
                                   C.byref(out)))
        return Cache(out.value, self)


class Cache(_Obj):
    _dtor = "rk_cache_destroy"

    def __init__(self, ptr, weights):
        super().__init__(ptr, weights)
        self.weights = weights

    @property
    def segment_len(self):
        return int(lib().rk_cache_segment_len(P(self.ptr)))

    def wait(self):
        """Block until an asynchronous upload has landed, deferred layers
        included (rk_cache_wait): the host arrays may be freed afterwards."""
        _check(lib().rk_cache_wait(P(self.ptr)))

    def xfer_wait(self):
        """Block until the copies issued so far have landed (deferred layers
        stay deferred) -- a diagnostic for timing the upload alone."""
        _check(lib().rk_cache_sync(P(self.ptr)))

    def save(self, path):
        """save_relay_cache (relay_cache.cpp:238-245): the RKRC file (rk_cache_save)."""
        _check(lib().rk_cache_save(P(self.ptr), os.fsencode(path)))

    def to_host(self):
        s = self.weights.spec
        n, L, kv, d = self.segment_len, s.num_layers, s.kv_dim, s.d_model
        toks = np.empty(n, np.int32)
        k = np.empty((L, n, kv), np.float32)
        v = np.empty((L, n, kv), np.float32)
        h = np.empty((n, d), np.float32)
        inf = np.empty(n, np.float32)
        kp = (F32P * L)(*[k[l].ctypes.data_as(F32P) for l in range(L)])
        vp = (F32P * L)(*[v[l].ctypes.data_as(F32P) for l in range(L)])
        src, snap = U64(), U64()
        _check(lib().rk_cache_export(P(self.ptr), toks.ctypes.data_as(I32P), kp, vp, h.ctypes.data_as(F32P),
                                     inf.ctypes.data_as(F32P), C.byref(src), C.byref(snap)))
        return HostRelayCache(num_kv_heads=s.num_kv_heads, d_head=s.d_head, d_model=d,
                              theta_base=s.theta_base, max_positions=s.max_positions,
                              segment_tokens=toks, source_base_position=src.value,
                              snapshot_layer=snap.value, k_pre=k, v=v, hidden_snapshot=h, influence=inf)


class Context(_Obj):
    """MergedKVContext on the device (KVContext rows [layer][pos][kv_dim] + SegmentMarks)."""
    _dtor = "rk_context_destroy"

    def __init__(self, ptr, weights):
        super().__init__(ptr, weights)
        self.weights = weights
        self.spec = weights.spec

    @property
    def size(self):
        return int(lib().rk_context_size(P(self.ptr)))

    def clone(self):
        out = P()
        _check(lib().rk_context_clone(P(self.ptr), C.byref(out)))
        return Context(out.value, self.weights)

    def reset(self):
        """Empty the context, keeping its device allocation."""
        _check(lib().rk_context_reset(P(self.ptr)))

    def export(self, layer, pos=0, count=None):
        kv = self.spec.kv_dim
        count = self.size - pos if count is None else count
        k = np.empty((count, kv), np.float32)
        v = np.empty((count, kv), np.float32)
        _check(lib().rk_context_export(P(self.ptr), U64(layer), U64(pos), U64(count),
                                       k.ctypes.data_as(F32P), v.ctypes.data_as(F32P)))
        return k, v

    def all(self):
        ks, vs = zip(*(self.export(l) for l in range(self.spec.num_layers)))
        return np.stack(ks), np.stack(vs)

    def segments(self):
        out = []
        L = self.spec.num_layers
        for i in range(int(lib().rk_context_num_segments(P(self.ptr)))):
            base, ln = U64(), U64()
            _check(lib().rk_context_segment(P(self.ptr), U64(i), C.byref(base), C.byref(ln), None))
            origin = np.empty(L * ln.value, np.uint8)
            _check(lib().rk_context_segment(P(self.ptr), U64(i), C.byref(base), C.byref(ln),
                                            origin.ctypes.data_as(C.POINTER(C.c_uint8))))
            out.append((base.value, ln.value, origin.reshape(L, ln.value)))
        return out

    # ---- hot path --------------------------------------------------------------
    def prefill(self, tokens, base=None, logits=True):
        """prefill (model.cpp:305-331); returns the last row's logits (or None)."""
        a, p = _i32(tokens)
        base = self.size if base is None else base
        out = np.empty(self.spec.vocab_size, np.float32) if logits else None
        w = self.weights
        _check(lib().rk_prefill(P(w.engine.ptr), P(w.ptr), P(self.ptr), p, U64(len(a)), U64(base),
                                out.ctypes.data_as(F32P) if logits else None))
        return out

    def relay_extend(self, cache, profile, opts, outputs=True):
        """relay_extend (relay_engine.cpp:183-361)."""
        w = self.weights
        o, bufs = _out_struct(self.spec, cache.segment_len, outputs)
        _check(lib().rk_relay_extend(P(w.engine.ptr), P(w.ptr), P(self.ptr), P(cache.ptr),
                                     C.byref(profile), C.byref(opts), C.byref(o)))
        return _out_dict(o, bufs)

    def relay_prefill(self, prefix, cache, profile, opts):
        """relay_prefill (relay_engine.cpp:363-395) into this (empty) context."""
        a, p = _i32(prefix)
        w = self.weights
        o, bufs = _out_struct(self.spec, cache.segment_len, True)
        logits = np.empty(self.spec.vocab_size, np.float32)
        _check(lib().rk_relay_prefill(P(w.engine.ptr), P(w.ptr), P(self.ptr), p, U64(len(a)), P(cache.ptr),
                                      C.byref(profile), C.byref(opts), C.byref(o), logits.ctypes.data_as(F32P)))
        d = _out_dict(o, bufs)
        d["logits"] = logits
        return d

    def agent_prefill(self, prefix, caches, suffix, profile, opts, want_logits=True, outputs=False):
        """run_workflow's downstream-agent TTFT sequence (workflow.cpp:316-369)."""
        a, p = _i32(prefix)
        s, sp = _i32(suffix)
        w = self.weights
        arr = (P * max(len(caches), 1))(*[c.ptr for c in caches])
        logits = np.empty(self.spec.vocab_size, np.float32) if want_logits else None
        tok = C.c_int32()
        outs = None
        bufs = []
        if outputs and caches:
            outs = (RelayOutput * len(caches))()
            for i, c in enumerate(caches):
                o, b = _out_struct(self.spec, c.segment_len, True)
                outs[i] = o
                bufs.append(b)
        _check(lib().rk_agent_prefill(P(w.engine.ptr), P(w.ptr), P(self.ptr), p, U64(len(a)), arr,
                                      U64(len(caches)), sp, U64(len(s)), C.byref(profile), C.byref(opts),
                                      outs, logits.ctypes.data_as(F32P) if want_logits else None,
                                      C.byref(tok)))
        res = {"logits": logits, "first_token": tok.value}
        if outs is not None:
            res["segments"] = [_out_dict(outs[i], bufs[i]) for i in range(len(caches))]
        return res

    def capture_prefill(self, tokens, snapshot_layer, include_self=False):
        a, p = _i32(tokens)
        w = self.weights
        out = P()
        _check(lib().rk_cache_capture_prefill(P(w.engine.ptr), P(w.ptr), P(self.ptr), p, U64(len(a)),
                                              U64(snapshot_layer), int(include_self), C.byref(out)))
        return Cache(out.value, w)

    def capture_decode(self, first_logits, n, snapshot_layer, include_self=False):
        w = self.weights
        fl = None
        if first_logits is not None:
            fl = np.ascontiguousarray(first_logits, np.float32)
        out = P()
        _check(lib().rk_cache_capture_decode(P(w.engine.ptr), P(w.ptr), P(self.ptr),
                                             fl.ctypes.data_as(F32P) if fl is not None else None, U64(n),
                                             U64(snapshot_layer), int(include_self), C.byref(out)))
        return Cache(out.value, w)


def _out_struct(spec, n, outputs=True):
    o = RelayOutput()
    if not outputs:
        return o, None
    bufs = {
        "selection": np.zeros(n, np.uint64), "tags": np.zeros(n, np.uint32),
        "s_dev": np.zeros(n, np.float64), "s_key_dev": np.zeros(n, np.float64),
        "hidden": np.zeros((n, spec.d_model), np.float32), "depth": np.zeros(n, np.uint64),
        "origin": np.zeros((spec.num_layers, n), np.uint8),
    }
    o.selection_indices = bufs["selection"].ctypes.data_as(C.POINTER(C.c_uint64))
    o.selection_tags = bufs["tags"].ctypes.data_as(C.POINTER(C.c_uint32))
    o.s_dev = bufs["s_dev"].ctypes.data_as(C.POINTER(C.c_double))
    o.s_key_dev = bufs["s_key_dev"].ctypes.data_as(C.POINTER(C.c_double))
    o.segment_hidden = bufs["hidden"].ctypes.data_as(F32P)
    o.hidden_depth = bufs["depth"].ctypes.data_as(C.POINTER(C.c_uint64))
    o.origin = bufs["origin"].ctypes.data_as(C.POINTER(C.c_uint8))
    return o, bufs


def _out_dict(o, bufs):
    d = {"segment_base": o.segment_base, "segment_len": o.segment_len,
         "selection_count": o.selection_count, "dev_threshold": o.dev_threshold,
         "min_dev_margin": o.min_dev_margin, "stats": stats_dict(o.stats)}
    if bufs is not None:
        k = o.selection_count
        d.update({
            "selection": bufs["selection"][:k].astype(np.int64), "tags": bufs["tags"][:k].copy(),
            "s_dev": bufs["s_dev"][:o.s_dev_len].copy(), "s_key_dev": bufs["s_key_dev"][:o.s_dev_len].copy(),
            "hidden": bufs["hidden"], "depth": bufs["depth"].astype(np.int64), "origin": bufs["origin"],
        })
    return d


def flops_span_full(spec, base, n):
    return lib().rk_flops_span_full(C.byref(spec), U64(base), U64(n))


def flops_segment_schedule(spec, base, n, lo, hi, sparse_hi, selected):
    return lib().rk_flops_segment_schedule(C.byref(spec), U64(base), U64(n), U64(lo), U64(hi),
                                           U64(sparse_hi), U64(selected))

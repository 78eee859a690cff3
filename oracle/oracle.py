"""Python access to the CHECKERS (test infrastructure only).

Two interchangeable CPU implementations of the reference relay-prefill path:

  Oracle("restatement")  build/liboracle.so   -- relay_oracle.c, the C
                         restatement (each function cites reference file:line)
  Oracle("reference")    _ref/librelaykv_ref.so -- the reference library itself,
                         compiled from /root/reference/proj/src (oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg /
--impl reference) may import this module. The product path never does.
"""
import ctypes as C
import os

import numpy as np

from paper_2603_13289_b200.abi import (LayerProfile, ModelSpec, RelayCacheView, RelayOptions,
                                       RelayOutput, exception_for, stats_dict)
from paper_2603_13289_b200.hostcache import HostRelayCache

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "restatement": os.path.join(HERE, "build", "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "librelaykv_ref.so"),
}

P = C.c_void_p
U64 = C.c_uint64
I32P = C.POINTER(C.c_int32)
F32P = C.POINTER(C.c_float)


def available(kind):
    return os.path.exists(LIB_PATHS[kind])


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(I32P)


class _Handle:
    def __init__(self, lib, ptr, dtor):
        self.ptr, self._lib, self._dtor = ptr, lib, dtor

    def __del__(self):
        try:
            if self.ptr:
                self._dtor(self.ptr)
                self.ptr = None
        except Exception:
            pass


class Oracle:
    def __init__(self, kind="restatement"):
        if kind not in LIB_PATHS:
            raise ValueError(kind)
        if not available(kind):
            raise FileNotFoundError(f"{LIB_PATHS[kind]} not built (run `make -C oracle`)")
        self.kind = kind
        self.lib = C.CDLL(LIB_PATHS[kind])
        self.pre = "ref_" if kind == "reference" else "orc_"
        L = self.lib
        getattr(L, self.pre + "last_error").restype = C.c_char_p
        for name in ("weights_tensor",):
            getattr(L, self.pre + name).restype = F32P
            getattr(L, self.pre + name).argtypes = [P, U64, C.POINTER(U64)]
        for name in ("ctx_size", "ctx_num_segments"):
            getattr(L, self.pre + name).restype = U64
            getattr(L, self.pre + name).argtypes = [P]
        getattr(L, self.pre + "flops_span_full").restype = C.c_double
        getattr(L, self.pre + "flops_span_full").argtypes = [C.POINTER(ModelSpec), U64, U64]
        getattr(L, self.pre + "flops_segment_schedule").restype = C.c_double
        getattr(L, self.pre + "flops_segment_schedule").argtypes = [C.POINTER(ModelSpec), U64, U64, U64, U64, U64, U64]
        fx = "ref_host_expf" if kind == "reference" else "orc_host_expf"
        getattr(L, fx).restype = C.c_float
        getattr(L, fx).argtypes = [C.c_float]
        self._expf = getattr(L, fx)
        if kind == "restatement":
            for name in ("weights_init", "ctx_create", "ctx_clone"):
                getattr(L, "orc_" + name).restype = P
            L.orc_weights_init.argtypes = [C.POINTER(ModelSpec), U64]
            L.orc_ctx_create.argtypes = [P]
            L.orc_ctx_clone.argtypes = [P]
            L.orc_mean_head_cosine_deviation.restype = C.c_double
            L.orc_mean_head_cosine_deviation.argtypes = [F32P, F32P, U64, U64]
        for name in ("weights_destroy", "ctx_destroy", "cache_destroy"):
            getattr(L, self.pre + name).argtypes = [P]
            getattr(L, self.pre + name).restype = None

    # ---- error handling -------------------------------------------------
    def _check(self, st):
        if st != 0:
            raise exception_for(st, getattr(self.lib, self.pre + "last_error")().decode())

    # ---- weights ----------------------------------------------------------
    def weights(self, spec, seed, checked=False):
        if self.kind == "reference":
            out = P()
            self._check(self.lib.ref_weights_create(C.byref(spec), U64(seed), int(checked), C.byref(out)))
            ptr = out.value
        else:
            ptr = self.lib.orc_weights_init(C.byref(spec), U64(seed))
        h = _Handle(self.lib, ptr, getattr(self.lib, self.pre + "weights_destroy"))
        h.spec = spec
        return h

    def weights_tensor(self, w, idx):
        n = U64()
        p = getattr(self.lib, self.pre + "weights_tensor")(P(w.ptr), U64(idx), C.byref(n))
        return np.ctypeslib.as_array(p, (n.value,)).copy()

    # ---- contexts -----------------------------------------------------------
    def new_ctx(self, w):
        if self.kind == "reference":
            out = P()
            self._check(self.lib.ref_ctx_create(P(w.ptr), C.byref(out)))
            ptr = out.value
        else:
            ptr = self.lib.orc_ctx_create(P(w.ptr))
        h = _Handle(self.lib, ptr, getattr(self.lib, self.pre + "ctx_destroy"))
        h.spec = w.spec
        return h

    def clone_ctx(self, ctx):
        if self.kind == "reference":
            out = P()
            self._check(self.lib.ref_ctx_clone(P(ctx.ptr), C.byref(out)))
            ptr = out.value
        else:
            ptr = self.lib.orc_ctx_clone(P(ctx.ptr))
        h = _Handle(self.lib, ptr, getattr(self.lib, self.pre + "ctx_destroy"))
        h.spec = ctx.spec
        return h

    def ctx_size(self, ctx):
        return int(getattr(self.lib, self.pre + "ctx_size")(P(ctx.ptr)))

    def ctx_export(self, ctx, layer, pos=0, count=None):
        kv = ctx.spec.kv_dim
        if count is None:
            count = self.ctx_size(ctx) - pos
        k = np.empty((count, kv), np.float32)
        v = np.empty((count, kv), np.float32)
        self._check(getattr(self.lib, self.pre + "ctx_export")(P(ctx.ptr), U64(layer), U64(pos), U64(count),
                                                      k.ctypes.data_as(F32P), v.ctypes.data_as(F32P)))
        return k, v

    def ctx_all(self, ctx):
        """[L, size, kv] K and V of the whole context."""
        ks, vs = zip(*(self.ctx_export(ctx, l) for l in range(ctx.spec.num_layers)))
        return np.stack(ks), np.stack(vs)

    def ctx_segments(self, ctx):
        segs = []
        for i in range(int(getattr(self.lib, self.pre + "ctx_num_segments")(P(ctx.ptr)))):
            base, ln = U64(), U64()
            self._check(getattr(self.lib, self.pre + "ctx_segment")(P(ctx.ptr), U64(i), C.byref(base), C.byref(ln), None))
            origin = np.empty(ctx.spec.num_layers * ln.value, np.uint8)
            self._check(getattr(self.lib, self.pre + "ctx_segment")(P(ctx.ptr), U64(i), C.byref(base), C.byref(ln),
                                                           origin.ctypes.data_as(C.POINTER(C.c_uint8))))
            segs.append((base.value, ln.value, origin.reshape(ctx.spec.num_layers, ln.value)))
        return segs

    # ---- model ---------------------------------------------------------------
    def prefill(self, w, ctx, tokens, base=None, logits=True):
        a, p = _i32(tokens)
        base = self.ctx_size(ctx) if base is None else base
        out = np.empty(w.spec.vocab_size, np.float32) if logits else None
        self._check(getattr(self.lib, self.pre + "prefill")(P(w.ptr), P(ctx.ptr), p, U64(len(a)), U64(base),
                                                   out.ctypes.data_as(F32P) if logits else None))
        return out

    def row_logits_from_layer(self, w, hidden_row, first_layer, ctx, position):
        h = np.ascontiguousarray(hidden_row, np.float32)
        out = np.empty(w.spec.vocab_size, np.float32)
        self._check(getattr(self.lib, self.pre + "row_logits_from_layer")(
            P(w.ptr), h.ctypes.data_as(F32P), U64(first_layer), P(ctx.ptr), U64(position),
            out.ctypes.data_as(F32P)))
        return out

    # ---- relay caches ---------------------------------------------------------
    def _cache_to_host(self, cptr):
        view = RelayCacheView()
        # ask for the layer count via a first view call with generous pointer arrays
        kp = (F32P * 4096)()
        vp = (F32P * 4096)()
        self._check(getattr(self.lib, self.pre + "cache_view")(P(cptr), C.byref(view), kp, vp))
        return HostRelayCache.from_view(view)

    def scenario(self, w, old_prefix, segment_len, snapshot_layer, include_self=False,
                 return_decode_ctx=False):
        """Decode segment_len tokens after old_prefix with capture (test_engine.cpp:43-62).
        Returns a HostRelayCache (and the decode-time context if asked)."""
        a, p = _i32(old_prefix)
        if self.kind == "reference":
            cache, dctx = P(), P()
            self._check(self.lib.ref_scenario_create(P(w.ptr), p, U64(len(a)), U64(segment_len),
                                                     U64(snapshot_layer), int(include_self),
                                                     C.byref(cache), C.byref(dctx)))
            host = self._cache_to_host(cache.value)
            self.lib.ref_cache_destroy(cache.value)
            ctx = _Handle(self.lib, dctx.value, self.lib.ref_ctx_destroy)
            ctx.spec = w.spec
        else:
            ctx = self.new_ctx(w)
            logits = self.prefill(w, ctx, a, 0, logits=True)
            cache = P()
            self._check(self.lib.orc_capture_decode(P(w.ptr), P(ctx.ptr), logits.ctypes.data_as(F32P),
                                                    U64(segment_len), U64(snapshot_layer),
                                                    int(include_self), C.byref(cache)))
            host = self._cache_to_host(cache.value)
            self.lib.orc_cache_destroy(cache.value)
        return (host, ctx) if return_decode_ctx else host

    def upload_cache(self, host):
        out = P()
        self._check(getattr(self.lib, self.pre + "cache_from_view")(C.byref(host.view()), C.byref(out)))
        return _Handle(self.lib, out.value, getattr(self.lib, self.pre + "cache_destroy"))

    def save_cache(self, host, path):
        """save_relay_cache (relay_cache.cpp:238-245) -- the reference library only."""
        assert self.kind == "reference", "RKRC files exist only in the reference build"
        c = self.upload_cache(host)
        self._check(self.lib.ref_cache_save(P(c.ptr), os.fsencode(path)))

    def load_cache(self, path):
        """load_relay_cache (relay_cache.cpp:247-253) -> HostRelayCache."""
        assert self.kind == "reference", "RKRC files exist only in the reference build"
        out = P()
        self._check(self.lib.ref_cache_load(os.fsencode(path), C.byref(out)))
        h = _Handle(self.lib, out.value, self.lib.ref_cache_destroy)
        return self._cache_to_host(h.ptr)

    # ---- offline profiler (reference library only) ---------------------------
    def profile_model(self, w, calib, params):
        from paper_2603_13289_b200.abi import ProfileResult
        assert self.kind == "reference"
        L = w.spec.num_layers
        out, s, rho = ProfileResult(), np.empty(L), np.empty(max(L - 1, 1))
        dp = C.POINTER(C.c_double)
        self._check(self.lib.ref_profile_model(P(w.ptr), C.byref(calib), C.byref(params), C.byref(out),
                                               s.ctypes.data_as(dp), rho.ctypes.data_as(dp)))
        d = out.as_dict()
        d["curve_s"], d["curve_rho"] = s, rho[:L - 1]
        return d

    def token_deviation(self, reuse_host, full_host):
        assert self.kind == "reference"
        a, b = self.upload_cache(reuse_host), self.upload_cache(full_host)
        L, n = reuse_host.num_layers, reuse_host.segment_len
        out = {k: np.empty((n, L), np.float64) for k in ("value_cos", "key_cos", "value_norm", "key_norm")}
        dp = C.POINTER(C.c_double)
        self._check(self.lib.ref_token_deviation(P(a.ptr), P(b.ptr), *[out[k].ctypes.data_as(dp) for k in
                                                                        ("value_cos", "key_cos", "value_norm",
                                                                         "key_norm")]))
        return out

    def layer_curve(self, value_cos):
        m = np.ascontiguousarray(value_cos, np.float64)
        n, L = m.shape
        s, rho, deg = np.empty(L), np.empty(L), np.empty(L, np.uint8)
        dp = C.POINTER(C.c_double)
        self._check(self.lib.ref_layer_curve(m.ctypes.data_as(dp), U64(n), U64(L), s.ctypes.data_as(dp),
                                             rho.ctypes.data_as(dp), deg.ctypes.data_as(C.POINTER(C.c_uint8))))
        return {"s": s, "rho": rho, "rho_degenerate": deg.astype(bool)}

    def average_curves(self, curves):
        s = np.ascontiguousarray([c["s"] for c in curves], np.float64)
        rho = np.ascontiguousarray([c["rho"] for c in curves], np.float64)
        deg = np.ascontiguousarray([c["rho_degenerate"] for c in curves], np.uint8)
        k, L = s.shape
        so, ro, do = np.empty(L), np.empty(L), np.empty(L, np.uint8)
        dp, up = C.POINTER(C.c_double), C.POINTER(C.c_uint8)
        self._check(self.lib.ref_average_curves(s.ctypes.data_as(dp), rho.ctypes.data_as(dp), deg.ctypes.data_as(up),
                                                U64(k), U64(L), so.ctypes.data_as(dp), ro.ctypes.data_as(dp),
                                                do.ctypes.data_as(up)))
        return {"s": so, "rho": ro, "rho_degenerate": do.astype(bool)}

    def profile_from_curve(self, curve, params):
        from paper_2603_13289_b200.abi import ProfileResult
        s = np.ascontiguousarray(curve["s"], np.float64)
        rho = np.ascontiguousarray(curve["rho"], np.float64)
        deg = np.ascontiguousarray(curve["rho_degenerate"], np.uint8)
        L = s.shape[0]
        out, crho = ProfileResult(), np.empty(max(L - 1, 1))
        dp = C.POINTER(C.c_double)
        self._check(self.lib.ref_profile_from_curve(s.ctypes.data_as(dp), rho.ctypes.data_as(dp),
                                                    deg.ctypes.data_as(C.POINTER(C.c_uint8)), U64(L),
                                                    C.byref(params), C.byref(out), crho.ctypes.data_as(dp)))
        d = out.as_dict()
        d["curve_s"], d["curve_rho"] = s, crho[:L - 1]
        return d

    def realign(self, host, base):
        c = self.upload_cache(host)
        L, n, kv = host.k_pre.shape
        out = np.empty((L, n, kv), np.float32)
        ptrs = (F32P * L)(*[out[l].ctypes.data_as(F32P) for l in range(L)])
        self._check(getattr(self.lib, self.pre + "realign")(P(c.ptr), U64(base), ptrs))
        return out

    # ---- hot path ---------------------------------------------------------------
    @staticmethod
    def _out_struct(spec, n):
        bufs = {
            "selection": np.zeros(n, np.uint64), "tags": np.zeros(n, np.uint32),
            "s_dev": np.zeros(n, np.float64), "s_key_dev": np.zeros(n, np.float64),
            "hidden": np.zeros((n, spec.d_model), np.float32), "depth": np.zeros(n, np.uint64),
            "origin": np.zeros((spec.num_layers, n), np.uint8),
        }
        o = RelayOutput()
        o.selection_indices = bufs["selection"].ctypes.data_as(C.POINTER(C.c_uint64))
        o.selection_tags = bufs["tags"].ctypes.data_as(C.POINTER(C.c_uint32))
        o.s_dev = bufs["s_dev"].ctypes.data_as(C.POINTER(C.c_double))
        o.s_key_dev = bufs["s_key_dev"].ctypes.data_as(C.POINTER(C.c_double))
        o.segment_hidden = bufs["hidden"].ctypes.data_as(F32P)
        o.hidden_depth = bufs["depth"].ctypes.data_as(C.POINTER(C.c_uint64))
        o.origin = bufs["origin"].ctypes.data_as(C.POINTER(C.c_uint8))
        return o, bufs

    @staticmethod
    def _out_dict(o, bufs):
        k = o.selection_count
        return {
            "selection": bufs["selection"][:k].astype(np.int64), "tags": bufs["tags"][:k].copy(),
            "s_dev": bufs["s_dev"][:o.s_dev_len].copy(), "s_key_dev": bufs["s_key_dev"][:o.s_dev_len].copy(),
            "hidden": bufs["hidden"], "depth": bufs["depth"].astype(np.int64), "origin": bufs["origin"],
            "segment_base": o.segment_base, "segment_len": o.segment_len,
            "dev_threshold": o.dev_threshold, "min_dev_margin": o.min_dev_margin,
            "stats": stats_dict(o.stats),
        }

    def relay_extend(self, w, ctx, host_cache, profile, opts):
        c = self.upload_cache(host_cache)
        o, bufs = self._out_struct(w.spec, host_cache.segment_len)
        self._check(getattr(self.lib, self.pre + "relay_extend")(P(w.ptr), P(ctx.ptr), P(c.ptr), C.byref(profile),
                                                        C.byref(opts), C.byref(o)))
        return self._out_dict(o, bufs)

    def relay_prefill(self, w, prefix, host_cache, profile, opts):
        """Returns (output dict with 'logits', merged ctx handle)."""
        a, p = _i32(prefix)
        c = self.upload_cache(host_cache)
        o, bufs = self._out_struct(w.spec, host_cache.segment_len)
        logits = np.empty(w.spec.vocab_size, np.float32)
        if self.kind == "reference":
            cptr = P()
            self._check(self.lib.ref_relay_prefill(P(w.ptr), p, U64(len(a)), P(c.ptr), C.byref(profile),
                                                   C.byref(opts), C.byref(o), logits.ctypes.data_as(F32P),
                                                   C.byref(cptr)))
            ctx = _Handle(self.lib, cptr.value, self.lib.ref_ctx_destroy)
            ctx.spec = w.spec
        else:
            ctx = self.new_ctx(w)
            self._check(self.lib.orc_relay_prefill(P(w.ptr), P(ctx.ptr), p, U64(len(a)), P(c.ptr),
                                                   C.byref(profile), C.byref(opts), C.byref(o),
                                                   logits.ctypes.data_as(F32P)))
        d = self._out_dict(o, bufs)
        d["logits"] = logits
        return d, ctx

    def agent_prefill(self, w, prefix, host_caches, suffix, profile, opts, ctx=None):
        """run_workflow relay-branch TTFT sequence; returns (end_logits, first_token, ctx)."""
        a, p = _i32(prefix)
        s, sp = _i32(suffix)
        cs = [self.upload_cache(h) for h in host_caches]
        arr = (P * max(len(cs), 1))(*[c.ptr for c in cs])
        ctx = ctx or self.new_ctx(w)
        logits = np.empty(w.spec.vocab_size, np.float32)
        tok = C.c_int32()
        self._check(getattr(self.lib, self.pre + "agent_prefill")(P(w.ptr), P(ctx.ptr), p, U64(len(a)), arr,
                                                         U64(len(cs)), sp, U64(len(s)), C.byref(profile),
                                                         C.byref(opts), logits.ctypes.data_as(F32P),
                                                         C.byref(tok)))
        return logits, tok.value, ctx

    def agent_prefill_parallel(self, w, threads, prefix, host_caches, suffix, profile, opts):
        """Reference CPU arm: `threads` independent sessions; returns wall ms."""
        assert self.kind == "reference"
        a, p = _i32(prefix)
        s, sp = _i32(suffix)
        cs = [self.upload_cache(h) for h in host_caches]
        arr = (P * max(len(cs), 1))(*[c.ptr for c in cs])
        toks = np.zeros(threads, np.int32)
        ms = C.c_double()
        self._check(self.lib.ref_agent_prefill_parallel(P(w.ptr), U64(threads), p, U64(len(a)), arr,
                                                        U64(len(cs)), sp, U64(len(s)), C.byref(profile),
                                                        C.byref(opts), toks.ctypes.data_as(I32P),
                                                        C.byref(ms)))
        return ms.value, toks

    # ---- misc ---------------------------------------------------------------------
    def flops_span_full(self, spec, base, n):
        return getattr(self.lib, self.pre + "flops_span_full")(C.byref(spec), U64(base), U64(n))

    def flops_segment_schedule(self, spec, base, n, lo, hi, sparse_hi, sel):
        return getattr(self.lib, self.pre + "flops_segment_schedule")(C.byref(spec), U64(base), U64(n), U64(lo),
                                                             U64(hi), U64(sparse_hi), U64(sel))

    def host_expf(self, x):
        return self._expf(C.c_float(x))

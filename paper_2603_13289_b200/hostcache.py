"""Host-side RelayCache (relay_cache.hpp:23-46) as numpy arrays.

Produces the rk_relay_cache_view the C ABI consumes (rk_cache_upload) and can
be built from any view (e.g. one exported by another library).
"""
import ctypes as C
import os

import numpy as np

from .abi import RelayCacheView


class HostRelayCache:
    """Numpy mirror of relaykv::RelayCache: k_pre/v [L, n, kv_dim] fp32 (keys
    pre-RoPE), hidden_snapshot [n, d_model], influence [n], segment_tokens [n]."""

    def __init__(self, *, num_kv_heads, d_head, d_model, theta_base, max_positions,
                 segment_tokens, source_base_position, snapshot_layer, k_pre, v,
                 hidden_snapshot, influence, decode_steps_observed=None):
        self.num_kv_heads = int(num_kv_heads)
        self.d_head = int(d_head)
        self.d_model = int(d_model)
        self.theta_base = float(theta_base)
        self.max_positions = int(max_positions)
        self.segment_tokens = np.ascontiguousarray(segment_tokens, dtype=np.int32)
        self.source_base_position = int(source_base_position)
        self.snapshot_layer = int(snapshot_layer)
        self.k_pre = np.ascontiguousarray(k_pre, dtype=np.float32)
        self.v = np.ascontiguousarray(v, dtype=np.float32)
        self.hidden_snapshot = np.ascontiguousarray(hidden_snapshot, dtype=np.float32)
        self.influence = np.ascontiguousarray(influence, dtype=np.float32)
        self.decode_steps_observed = (len(self.segment_tokens) if decode_steps_observed is None
                                      else int(decode_steps_observed))
        self._keep = None

    @property
    def segment_len(self):
        return int(self.segment_tokens.shape[0])

    @property
    def num_layers(self):
        return int(self.k_pre.shape[0])

    def view(self):
        """rk_relay_cache_view pointing into this object's arrays (kept alive by self).
        Array shapes are checked first (the C ABI reads L x n x kv_dim floats per
        K/V table, n x d_model hidden floats and n influence scores); the
        reference's semantic checks (relay_cache.cpp:18-49) run in the ABI."""
        from paper_2603_13289_b200.abi import RK_ERR_INVALID_ARGUMENT, exception_for
        L, n, kv = self.num_layers, self.segment_len, self.num_kv_heads * self.d_head
        if self.k_pre.ndim != 3 or self.k_pre.shape[1:] != (n, kv) or self.v.shape != self.k_pre.shape:
            raise exception_for(RK_ERR_INVALID_ARGUMENT, "relay cache: K/V tables must be [L, n, kv_dim] "
                                f"({L}, {n}, {kv}); got {self.k_pre.shape} / {self.v.shape}")
        if self.hidden_snapshot.shape != (n, self.d_model):
            raise exception_for(RK_ERR_INVALID_ARGUMENT, "relay cache: hidden snapshot shape mismatch")
        if self.influence.shape != (n,):
            raise exception_for(RK_ERR_INVALID_ARGUMENT, "relay cache: influence length mismatch")
        kp = (C.POINTER(C.c_float) * max(L, 1))()
        vp = (C.POINTER(C.c_float) * max(L, 1))()
        for l in range(L):
            kp[l] = self.k_pre[l].ctypes.data_as(C.POINTER(C.c_float))
            vp[l] = self.v[l].ctypes.data_as(C.POINTER(C.c_float))
        v = RelayCacheView(
            L, self.num_kv_heads, self.d_head, self.d_model, self.theta_base, self.max_positions,
            self.segment_len, self.segment_tokens.ctypes.data_as(C.POINTER(C.c_int32)),
            self.source_base_position, self.snapshot_layer, self.decode_steps_observed,
            C.cast(kp, C.POINTER(C.POINTER(C.c_float))), C.cast(vp, C.POINTER(C.POINTER(C.c_float))),
            self.hidden_snapshot.ctypes.data_as(C.POINTER(C.c_float)),
            self.influence.ctypes.data_as(C.POINTER(C.c_float)))
        self._keep = (kp, vp, v)
        return v

    @classmethod
    def from_view(cls, v):
        L, n = int(v.num_layers), int(v.segment_len)
        kv = int(v.num_kv_heads * v.d_head)
        d = int(v.d_model)
        k_pre = np.stack([np.ctypeslib.as_array(v.k_pre[l], (n * kv,)).reshape(n, kv).copy()
                          for l in range(L)]) if n else np.zeros((L, 0, kv), np.float32)
        vv = np.stack([np.ctypeslib.as_array(v.v[l], (n * kv,)).reshape(n, kv).copy()
                       for l in range(L)]) if n else np.zeros((L, 0, kv), np.float32)
        return cls(num_kv_heads=v.num_kv_heads, d_head=v.d_head, d_model=d,
                   theta_base=v.theta_base, max_positions=v.max_positions,
                   segment_tokens=np.ctypeslib.as_array(v.segment_tokens, (n,)).copy() if n else [],
                   source_base_position=v.source_base_position, snapshot_layer=v.snapshot_layer,
                   k_pre=k_pre, v=vv,
                   hidden_snapshot=np.ctypeslib.as_array(v.hidden_snapshot, (n * d,)).reshape(n, d).copy()
                   if n else np.zeros((0, d), np.float32),
                   influence=np.ctypeslib.as_array(v.influence, (n,)).copy() if n else [],
                   decode_steps_observed=v.decode_steps_observed)

    def copy(self):
        return HostRelayCache(
            num_kv_heads=self.num_kv_heads, d_head=self.d_head, d_model=self.d_model,
            theta_base=self.theta_base, max_positions=self.max_positions,
            segment_tokens=self.segment_tokens.copy(), source_base_position=self.source_base_position,
            snapshot_layer=self.snapshot_layer, k_pre=self.k_pre.copy(), v=self.v.copy(),
            hidden_snapshot=self.hidden_snapshot.copy(), influence=self.influence.copy(),
            decode_steps_observed=self.decode_steps_observed)

    def save(self, path):
        """save_relay_cache (relay_cache.cpp:238-245) on the host: the RKRC
        file, byte-identical to the reference's (rk_cache_file_write)."""
        from .engine import _check, lib
        _check(lib().rk_cache_file_write(C.byref(self.view()), os.fsencode(path)))

    @classmethod
    def load(cls, path):
        """load_relay_cache (relay_cache.cpp:247-253) on the host: validates the
        container and the cache like the reference (rk_cache_file_read)."""
        from .engine import _check, lib
        h, v = C.c_void_p(), RelayCacheView()
        _check(lib().rk_cache_file_read(os.fsencode(path), C.byref(h), C.byref(v)))
        try:
            return cls.from_view(v)
        finally:
            lib().rk_cache_file_free(h)

    def to_bytes(self):
        """export_relay_cache (relay_cache.cpp:176-201): the RKRC bytes."""
        from .engine import _check, lib
        size = C.c_uint64()
        v = self.view()
        _check(lib().rk_cache_file_encode(C.byref(v), None, C.c_uint64(0), C.byref(size)))
        buf = (C.c_uint8 * size.value)()
        _check(lib().rk_cache_file_encode(C.byref(v), buf, size, C.byref(size)))
        return bytes(buf)

    @classmethod
    def from_bytes(cls, data):
        """import_relay_cache (relay_cache.cpp:203-236)."""
        from .engine import _check, lib
        data = bytes(data)
        h, v = C.c_void_p(), RelayCacheView()
        _check(lib().rk_cache_file_decode(C.c_char_p(data), C.c_uint64(len(data)), C.byref(h), C.byref(v)))
        try:
            return cls.from_view(v)
        finally:
            lib().rk_cache_file_free(h)

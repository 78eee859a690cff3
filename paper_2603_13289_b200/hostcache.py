"""Host-side RelayCache (relay_cache.hpp:23-46) as numpy arrays.

Produces the rk_relay_cache_view the C ABI consumes (rk_cache_upload) and can
be built from any view (e.g. one exported by another library).
"""
import ctypes as C

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
        """rk_relay_cache_view pointing into this object's arrays (kept alive by self)."""
        L = self.num_layers
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

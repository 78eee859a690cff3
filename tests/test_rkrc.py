"""RKRC relay-cache files (relay_cache.cpp:176-253, serialize.cpp:45-117) on the
host: the engine's codec (rk_cache_file_write / rk_cache_file_read) against the
golden files the reference wrote (tests/golden/make_rkrc.py) and, where
oracle/_ref is built, against the reference's save/load on random caches.
Mirrors the reference's test_relay_cache.cpp / test_serialization.cpp cases:
round trip, truncated header / manifest / blob, bad magic, bad version,
checksum mismatch, missing tensor, shape mismatch, negative influence,
unreadable path."""
import glob
import json
import os
import struct

import numpy as np
import pytest

from paper_2603_13289_b200.abi import InvalidArgument, IoError, SchemaError
from paper_2603_13289_b200.hostcache import HostRelayCache

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.rkrc")))


def ref_oracle():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    return Oracle("reference")


def fnv1a64(b):
    h = 0xcbf29ce484222325
    for x in b:
        h = ((h ^ x) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def split(data):
    mlen = struct.unpack_from("<Q", data, 8)[0]
    return data[:16], json.loads(data[16:16 + mlen]), data[16 + mlen:]


def join(manifest, blob, fix_checksum=True, version=1, magic=b"RKRC"):
    if fix_checksum:
        manifest = dict(manifest, blob_bytes=len(blob), blob_checksum=fnv1a64(blob))
    m = json.dumps(manifest, separators=(",", ":"), sort_keys=True).encode()
    return magic + struct.pack("<IQ", version, len(m)) + m + blob


def random_cache(seed, L=3, n=7, hkv=2, dh=4, d=16, theta=10000.0):
    r = np.random.default_rng(seed)
    return HostRelayCache(
        num_kv_heads=hkv, d_head=dh, d_model=d, theta_base=theta, max_positions=4096,
        segment_tokens=r.integers(0, 1000, n), source_base_position=int(r.integers(0, 500)),
        snapshot_layer=int(r.integers(0, L)), k_pre=r.standard_normal((L, n, hkv * dh)),
        v=r.standard_normal((L, n, hkv * dh)), hidden_snapshot=r.standard_normal((n, d)),
        influence=r.random(n), decode_steps_observed=n + int(r.integers(0, 3)))


def same(a, b):
    for f in ("num_kv_heads", "d_head", "d_model", "max_positions", "source_base_position", "snapshot_layer",
              "decode_steps_observed", "num_layers", "segment_len"):
        assert getattr(a, f) == getattr(b, f), f
    assert np.float32(a.theta_base) == np.float32(b.theta_base)
    for f in ("segment_tokens", "k_pre", "v", "hidden_snapshot", "influence"):
        x, y = getattr(a, f), getattr(b, f)
        assert x.shape == y.shape and x.tobytes() == y.tobytes(), f


def test_golden_files_present():
    assert len(GOLDEN) >= 2


@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_golden_roundtrip_byte_identical(path, tmp_path):
    """Reference-written file -> our reader -> our writer == the same bytes."""
    c = HostRelayCache.load(path)
    meta = json.load(open(path + ".json"))
    assert c.segment_len == meta["segment_len"] and c.snapshot_layer == meta["snapshot_layer"]
    assert c.source_base_position == len(meta["old_prefix"])
    out = tmp_path / "again.rkrc"
    c.save(out)
    assert out.read_bytes() == open(path, "rb").read()


@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_golden_matches_reference_loader(path):
    orc = ref_oracle()
    same(HostRelayCache.load(path), orc.load_cache(path))


@pytest.mark.parametrize("seed,theta", [(0, 10000.0), (1, 500000.0), (2, 1e6), (3, 12345.678), (4, 0.1),
                                        (5, 1.5e-7), (6, 3.4e38)])
def test_random_caches_byte_identical_to_reference(seed, theta, tmp_path):
    """Our writer == reference save_relay_cache byte for byte (incl. the
    manifest's float formatting), and each side loads the other's file."""
    orc = ref_oracle()
    c = random_cache(seed, L=1 + seed % 4, n=1 + 3 * seed, theta=theta)
    ours, theirs = tmp_path / "ours.rkrc", tmp_path / "theirs.rkrc"
    c.save(ours)
    orc.save_cache(c, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    same(orc.load_cache(ours), c)
    same(HostRelayCache.load(theirs), c)


def test_manifest_layout():
    data = open(GOLDEN[0], "rb").read()
    hdr, m, blob = split(data)
    assert hdr[:4] == b"RKRC" and struct.unpack_from("<I", hdr, 4)[0] == 1
    assert m["kind"] == "relay-cache" and m["schema_version"] == 1
    assert m["blob_bytes"] == len(blob) and m["blob_checksum"] == fnv1a64(blob)
    L = m["num_layers"]
    names = [t["name"] for t in m["tensors"]]
    assert names == sum([[f"k_pre.{l}", f"v.{l}"] for l in range(L)], []) + ["hidden_snapshot", "influence"]


def corruptions():
    data = open(GOLDEN[0], "rb").read()
    hdr, m, blob = split(data)
    flipped = bytearray(blob)
    flipped[5] ^= 1
    bad_inf = bytearray(blob)
    off = next(t["offset"] for t in m["tensors"] if t["name"] == "influence")
    bad_inf[off:off + 4] = struct.pack("<f", -1.0)
    no_hidden = dict(m, tensors=[t for t in m["tensors"] if t["name"] != "hidden_snapshot"])
    bad_shape = dict(m, tensors=[dict(t, shape=[t["shape"][0], t["shape"][1] + 1]) if t["name"] == "v.3" else t
                                 for t in m["tensors"]])
    past_end = dict(m, tensors=[dict(t, offset=len(blob)) if t["name"] == "influence" else t for t in m["tensors"]])
    snap_oob = dict(m, snapshot_layer=m["num_layers"])
    return {
        "truncated_header": data[:10],
        "bad_magic": b"RKWT" + data[4:],
        "bad_version": join(m, blob, version=2),
        "truncated_manifest": data[:16 + 20],
        "truncated_blob": data[:-8],
        "checksum": hdr + data[16:len(data) - len(blob)] + bytes(flipped),
        "manifest_garbage": b"RKRC" + struct.pack("<IQ", 1, 5) + b"{{{{{" + blob,
        "missing_tensor": join(no_hidden, blob),
        "shape_mismatch": join(bad_shape, blob),
        "past_end": join(past_end, blob),
        "negative_influence": join(m, bytes(bad_inf)),
        "snapshot_out_of_range": join(snap_oob, blob),
        "missing_key": join({k: v for k, v in m.items() if k != "d_model"}, blob),
    }


@pytest.mark.parametrize("kind", sorted(corruptions()))
def test_corrupt_files_raise_schema_error(kind, tmp_path):
    p = tmp_path / f"{kind}.rkrc"
    p.write_bytes(corruptions()[kind])
    with pytest.raises(SchemaError):
        HostRelayCache.load(p)


@pytest.mark.parametrize("kind", sorted(corruptions()))
def test_corrupt_files_same_status_as_reference(kind, tmp_path):
    orc = ref_oracle()
    p = tmp_path / f"{kind}.rkrc"
    p.write_bytes(corruptions()[kind])
    with pytest.raises(SchemaError) as ours:
        HostRelayCache.load(p)
    with pytest.raises(SchemaError) as theirs:
        orc.load_cache(p)
    if kind not in ("manifest_garbage", "missing_key"):  # nlohmann's own wording differs
        assert str(ours.value).split("] ", 1)[1] == str(theirs.value).split("] ", 1)[1]


def test_io_errors(tmp_path):
    with pytest.raises(IoError):
        HostRelayCache.load(tmp_path / "does_not_exist.rkrc")
    with pytest.raises(IoError):
        random_cache(0).save(tmp_path / "no_such_dir" / "x.rkrc")
    assert issubclass(IoError, OSError)


def test_save_validates_like_export(tmp_path):
    c = random_cache(1)
    c.influence[2] = -0.5
    with pytest.raises(InvalidArgument):
        c.save(tmp_path / "x.rkrc")
    assert not (tmp_path / "x.rkrc").exists()


@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_bytes_api_matches_file_api(path):
    """export_relay_cache / import_relay_cache on byte buffers (test_relay_cache.cpp:251-276)."""
    data = open(path, "rb").read()
    c = HostRelayCache.from_bytes(data)
    same(c, HostRelayCache.load(path))
    assert c.to_bytes() == data
    with pytest.raises(SchemaError):
        HostRelayCache.from_bytes(data[:-3])
    with pytest.raises(SchemaError):
        HostRelayCache.from_bytes(b"")


def test_theta_float_formatting_sweep_matches_reference(tmp_path):
    """nlohmann::json dump formats the manifest's theta_base with Grisu2
    (shortest digits in most cases, not all); the engine's formatter searches
    the shortest round-trip digits. A randomized sweep of float theta values
    over 80 binades pins that both produce the same bytes."""
    orc = ref_oracle()
    r = np.random.default_rng(7)
    exps = r.integers(-40, 40, 1500)
    mant = r.random(1500) + 1.0
    thetas = [float(np.float32(m * 2.0 ** int(e))) for m, e in zip(mant, exps)]
    thetas += [float(np.float32(x)) for x in (1e4, 5e5, 1e6, 1e-3, 123456.789, 3.0e38, 1.17549435e-38)]
    base = random_cache(11, L=1, n=1)
    ours, theirs = tmp_path / "o.rkrc", tmp_path / "t.rkrc"
    bad = []
    for th in thetas:
        base.theta_base = th
        base.save(ours)
        orc.save_cache(base, theirs)
        a, b = ours.read_bytes(), theirs.read_bytes()
        if a != b:
            bad.append((th, split(a)[1].get("theta_base"), split(b)[1].get("theta_base")))
    assert not bad, bad[:10]


def test_view_rejects_malformed_arrays():
    """HostRelayCache.view() checks array shapes before handing pointers to
    the C ABI (which reads L x n x kv_dim floats per table): a short V table,
    a wrong hidden snapshot or influence length is InvalidArgument, not a
    heap over-read."""
    for mutate in (lambda c: setattr(c, "v", np.ascontiguousarray(c.v[:, :2])),
                   lambda c: setattr(c, "hidden_snapshot", np.ascontiguousarray(c.hidden_snapshot[:, :3])),
                   lambda c: setattr(c, "influence", np.ascontiguousarray(c.influence[:1]))):
        c = random_cache(5, L=2, n=4)
        mutate(c)
        with pytest.raises(InvalidArgument):
            c.view()

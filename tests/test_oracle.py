"""CPU tests: the C restatement (oracle/fpx_oracle.c) pinned against the
reference's golden vectors (tests/golden/, generated from the unmodified
reference by make_golden.py), the SPEC known answers and the
SPEC acceptance criteria."""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")

from tests.golden.make_golden import FULL, activations, weights  # noqa: E402
from oracle.oracle import split_for  # noqa: E402


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLD, "golden.json")) as f:
        meta = json.load(f)
    return meta, np.load(os.path.join(GOLD, "golden.npz"))


# ------------------------------------------------------------ scalar KATs
def test_spec_decode_kats(oracle):
    # SPEC.md:58-68 (with the 0b011100 erratum: 1.0 is 0b001100)
    assert oracle.decode(0b000000, 3, 2) == 0.0
    assert oracle.decode(0b001100, 3, 2) == 1.0
    assert oracle.decode(0b011100, 3, 2) == 16.0
    assert oracle.decode(0b011111, 3, 2) == 28.0
    assert oracle.decode(0b000001, 3, 2) == 0.0625
    # SPEC.md:69-70
    assert oracle.encode(1000.0, 3, 2) == 0b011111
    assert oracle.encode(-0.0, 3, 2) == 0b100000
    assert oracle.encode(1.0, 3, 2) == 0b001100


def test_spec_half_and_scale_kats(oracle):
    # eff scale of 1.0 is 4096; 0x0C00 * 4096 = 1.0; 0x8C00 -> -1.0
    assert oracle.effective_scale(0x3C00, 3, 2) == 0x6C00
    assert oracle.half_mul(0x0C00, 0x6C00) == 0x3C00
    assert oracle.half_mul(0x8C00, 0x6C00) == 0xBC00
    # code 0.0625 at scale 2.0 -> 0.125
    assert oracle.half_mul(oracle.float_to_half(oracle.decode(1, 3, 2)), 0x4000) == 0x3000


def test_kat_tables_match_reference(oracle, golden):
    meta, _ = golden
    for name, kat in meta["kat"].items():
        if not name.startswith("e") or "m" not in name or len(name) != 4:
            continue
        e, m = int(name[1]), int(name[3])
        for c, v in enumerate(kat["decode"]):
            assert oracle.decode(c, e, m) == v, (name, c)
        assert kat["encode_roundtrip"] == list(range(1 << (1 + e + m))), name
        for c in range(1 << (1 + e + m)):
            assert oracle.encode(oracle.decode(c, e, m), e, m) == c
        for s, eff in kat["effective_scale"].items():
            assert oracle.effective_scale(int(s), e, m) == eff, (name, s)
    for fmt, pairs in meta["kat"]["encode_samples"].items():
        e, m = int(fmt[1]), int(fmt[3])
        for v, code in pairs:
            assert oracle.encode(v, e, m) == code, (fmt, v)
    for a, b, r in meta["kat"]["half_mul"]:
        assert oracle.half_mul(a, b) == r


def test_half_roundtrip_exhaustive(oracle):
    for h in range(0, 1 << 16, 7):
        f = oracle.half_to_float(h)
        if f == f:  # not NaN
            assert oracle.float_to_half(f) == h


# ------------------------------------------------------------ golden cases
def test_small_cases_bit_exact(oracle, golden):
    meta, npz = golden
    for case in meta["cases"]:
        tag, e, m = case["tag"], case["e"], case["m"]
        w = weights(case["seed"], case["rows"], case["cols"])
        st, codes, scales, _ = oracle.quantize(w, e, m)
        assert st == 0
        assert (codes == npz[f"{tag}/codes"]).all(), tag
        assert (scales == npz[f"{tag}/scales"]).all(), tag
        st, streams = oracle.pack(codes, scales, e, m)
        assert st == 0
        for i, s in enumerate(streams):
            assert (s == npz[f"{tag}/stream{i}"]).all(), (tag, i)
        st, back = oracle.unpack(streams, *codes.shape, e, m)
        assert (back == codes).all()
        assert (oracle.dequantize(codes, scales, e, m) == npz[f"{tag}/dequant"]).all(), tag
        if (e, m) == (3, 2):  # Algorithm 1 on the packed words == scalar oracle
            assert (oracle.dequant_packed_e3m2(streams, scales, *codes.shape) == npz[f"{tag}/dequant"]).all()
        for n in case["batches"]:
            b = activations(case["seed"], n, case["cols"]).view(np.uint16)
            st, c = oracle.gemm_reference(codes, scales, e, m, b, orig_cols=case["cols"])
            assert st == 0
            assert (c.view(np.uint32) == npz[f"{tag}/C_n{n}"].view(np.uint32)).all(), (tag, n)


def test_full_size_4096_pins(oracle, golden):
    meta, _ = golden
    pin = [f for f in meta["full"] if f["rows"] == 4096][0]
    w = weights(pin["seed"], 4096, 4096)
    st, codes, scales, _ = oracle.quantize(w, 3, 2)
    assert st == 0
    assert oracle.fnv1a64(codes) == pin["codes_fnv"]
    assert oracle.fnv1a64(scales) == pin["scales_fnv"]
    st, streams = oracle.pack(codes, scales, 3, 2)
    assert [oracle.fnv1a64(s) for s in streams] == pin["streams_fnv"]


# ------------------------------------------------------ SPEC acceptance
def test_acceptance_1_exhaustive_codes_x_scales(oracle):
    """64 e3m2 codes x scales: Algorithm-1 word path == scalar oracle."""
    import ctypes as C
    for scale in (0x3C00, 0x3800, 0x4200, 0x0400, 0x0001, 0x4BFF):
        eff = oracle.effective_scale(scale, 3, 2)
        for code in range(64):
            # one thread's slice filled with the same code: build words via the
            # [2,4] split layout (all groups/lanes identical)
            hi2, lo4 = code >> 4, code & 0xF
            w2 = 0
            for lane in range(4):
                for g in range(4):
                    w2 |= hi2 << (8 * lane + 6 - 2 * g)
            w4 = 0
            for lane in range(4):
                for g in range(2):
                    w4 |= lo4 << (8 * lane + 4 - 4 * g)
            f1 = (C.c_uint32 * 2)(w2, w2)
            f2 = (C.c_uint32 * 4)(w4, w4, w4, w4)
            sc = (C.c_uint16 * 8)(*([eff] * 8))
            out = (C.c_uint16 * 32)()
            oracle.lib.orc_swar_thread_slice(f1, f2, sc, out)
            want = oracle.half_mul(oracle.float_to_half(oracle.decode(code, 3, 2)), scale)
            assert all(o == want for o in out), (hex(scale), code)


def test_acceptance_2_pack_unpack_roundtrip(oracle):
    rng = np.random.default_rng(5)
    for i in range(24):
        e, m = [(3, 2), (2, 3), (2, 2), (2, 1), (4, 3)][i % 5]
        rows, cols = (int(x) * 64 for x in rng.integers(1, 5, size=2))
        codes = rng.integers(0, 1 << (1 + e + m), size=(rows, cols), dtype=np.uint8)
        scales = np.full(rows, 0x3C00, np.uint16)
        st, streams = oracle.pack(codes, scales, e, m)
        assert st == 0
        assert sum(s.size for s in streams) * 8 == rows * cols * (1 + e + m)  # size law
        st, back = oracle.unpack(streams, rows, cols, e, m)
        assert (back == codes).all()


def test_acceptance_4_compression_ratio():
    # 4096^2: streams alone = 0.375 of fp16, with scales + header < 0.40
    streams = 4096 * 4096 * 6 // 8
    assert streams / (4096 * 4096 * 2) == 0.375
    assert (streams + 4096 * 2 + 64) / (4096 * 4096 * 2) < 0.40


def test_acceptance_6_eq3_identity(oracle):
    # decode(c) == new_cast(c) * 2^12 for all 64 codes
    for c in range(64):
        x = (c << 2)  # code at bits [7:2] of a byte lane
        v = (x & 0x80) | ((x >> 2) & 0x1F)  # dequant4 on one lane -> fp16 top byte
        h = v << 8
        assert oracle.half_to_float(h) * 4096.0 == oracle.decode(c, 3, 2)


def test_acceptance_8_quantization_error_bound(oracle):
    rng = np.random.default_rng(8)
    for e, m in [(3, 2), (2, 3), (2, 2)]:
        w = (rng.standard_normal((8, 1024)) * rng.uniform(0.01, 3.0, size=(8, 1))).astype(np.float32)
        st, codes, scales, _ = oracle.quantize(w, e, m)
        assert st == 0
        maxrep = oracle.lib.orc_max_rep(e, m)
        bias = (1 << (e - 1)) - 1
        for r in range(8):
            s = oracle.half_to_float(int(scales[r]))
            for c in range(0, 1024, 3):
                v = float(w[r, c])
                q = oracle.decode(int(codes[r, c]), e, m)
                a = abs(v / s)
                if a <= maxrep:
                    ex = max(int(np.floor(np.log2(a))) if a > 0 else 1 - bias, 1 - bias)
                    ulp = 2.0 ** (min(ex, (1 << e) - 1 - bias) - m)
                    assert abs(v - s * q) <= s * ulp / 2 * (1 + 1e-6) + 1e-30, (e, m, r, c)


def test_quantize_errors(oracle):
    w = np.ones((4, 64), np.float32)
    w[2, 5] = np.nan
    w[3, 0] = np.nan
    st, _, _, row = oracle.quantize(w, 3, 2)
    assert st == 3 and row == 2  # InvalidValue, first failing row
    big = np.full((2, 64), 1e9, np.float32)
    st, _, _, row = oracle.quantize(big, 3, 2)
    assert st == 4 and row == 0  # ScaleOverflow
    z = np.zeros((3, 70), np.float32)
    st, codes, scales, _ = oracle.quantize(z, 3, 2)
    assert st == 0 and (codes == 0).all() and (scales == 0x3C00).all()


def test_oracle_matches_reference_random(oracle, reference):
    """Extra random shapes / formats against the live reference build."""
    rng = np.random.default_rng(77)
    for e, m in [(3, 2), (2, 3), (2, 2), (2, 1), (3, 1), (4, 3)]:
        rows, cols = int(rng.integers(1, 200)), int(rng.integers(1, 300))
        w = (rng.standard_normal((rows, cols)) * rng.uniform(1e-3, 10)).astype(np.float32)
        st1, c1, s1, _ = oracle.quantize(w, e, m)
        st2, c2, s2 = reference.quantize(w, e, m)
        assert st1 == st2 == 0
        assert (c1 == c2).all() and (s1 == s2).all()
        st1, p1 = oracle.pack(c1, s1, e, m)
        st2, p2 = reference.pack(c2, s2, e, m, rows, cols)
        assert all((a == b).all() for a, b in zip(p1, p2))
        n = int(rng.integers(1, 20))
        b = rng.standard_normal((n, cols)).astype(np.float16).view(np.uint16)
        st, c_o = oracle.gemm_reference(c1, s1, e, m, b, orig_cols=cols)
        c_r = reference.prepare(c1, s1, e, m, rows, cols).gemm_reference(b)
        assert (c_o.view(np.uint32) == c_r.view(np.uint32)).all()


def test_split_presets():
    assert split_for(3, 2) == [2, 4] and split_for(2, 2) == [4, 1] and split_for(2, 1) == [4]
    assert split_for(1, 1) == [2, 1] and split_for(4, 2) == [4, 2, 1] and split_for(4, 3) == [4, 4]
    assert FULL[1][1:] == (8192, 22016)

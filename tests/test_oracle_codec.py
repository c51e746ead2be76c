"""Pins for the oracle's scalar codec (C1 decode, C2 encode, C3 scale, C5 shift).

Every check here compares the oracle with something other than itself: library routines
(torch.float8_e4m3fn, ml_dtypes.float8_e4m3fn), exact rational / integer arithmetic written
independently in Python, closed forms printed in the paper, and worked examples.
"""
import json
import math
import os

import ml_dtypes
import numpy as np
import pytest
import torch

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def torch_decode_table():
    return torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()


def torch_encode_f32(vals: np.ndarray) -> np.ndarray:
    """Library RNE cast fp32 -> E4M3 (torch CPU).  Only valid for |v| <= 448 (torch does not
    saturate: 500 -> NaN), which is the only range the method produces (C3 guarantees it)."""
    t = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float32))
    return t.to(torch.float8_e4m3fn).view(torch.uint8).numpy()


# ---------------------------------------------------------------------------------- C1 decode
def test_decode_matches_two_libraries(orc):
    o = orc.decode_table()
    t = torch_decode_table()
    m = np.arange(256, dtype=np.uint8).view(ml_dtypes.float8_e4m3fn).astype(np.float64)
    nan = np.isnan(o)
    assert np.array_equal(nan, np.isnan(t)) and np.array_equal(nan, np.isnan(m))
    assert set(np.nonzero(nan)[0].tolist()) == {0x7F, 0xFF}      # the only NaN codes, no Inf
    assert np.array_equal(o[~nan], t[~nan]) and np.array_equal(o[~nan], m[~nan])


def test_decode_paper_constants(orc):
    # P:143 "448 is the maximum representable number of FP8_E4M3"
    finite = [orc.decode_e4m3(c) for c in range(256) if c not in (0x7F, 0xFF)]
    assert max(finite) == 448.0 and orc.decode_e4m3(0x7E) == 448.0
    # Eq. 10 with SN=0, E=7, M=0 -> 2^0 * 1 = 1.0 ; smallest subnormal 2^-9
    assert orc.decode_e4m3(0x38) == 1.0
    assert orc.decode_e4m3(0x01) == 2.0 ** -9
    assert orc.decode_e4m3(0x80) == 0.0 and math.copysign(1, orc.decode_e4m3(0x80)) == -1


# ---------------------------------------------------------------------------------- C2 encode
def _probe_values():
    t = torch_decode_table()
    fin = np.sort(np.unique(t[(~np.isnan(t)) & (t >= 0)]))
    mids = (fin[:-1] + fin[1:]) / 2                                  # exact in fp32 (5 sig. bits)
    rng = np.random.default_rng(0)
    rand = np.concatenate([rng.uniform(-448, 448, 20000), rng.standard_normal(20000) * 0.01,
                           np.exp(rng.uniform(-25, 6, 20000)) * rng.choice([-1, 1], 20000)])
    near = np.concatenate([np.nextafter(mids.astype(np.float32), np.float32(0)),
                           np.nextafter(mids.astype(np.float32), np.float32(1000))]).astype(np.float64)
    v = np.concatenate([fin, -fin, mids, -mids, rand, near, -near]).astype(np.float32)
    return v[np.abs(v) <= 448.0]


def test_encode_matches_library_rne(orc):
    v = _probe_values()
    lib_codes = torch_encode_f32(v)
    ours = np.array([orc.encode_e4m3(float(x)) for x in v], dtype=np.uint8)
    bad = np.nonzero(ours != lib_codes)[0]
    assert bad.size == 0, [(float(v[i]), int(ours[i]), int(lib_codes[i])) for i in bad[:10]]


def test_encode_signed_zero_and_saturation(orc):
    # R10: the sign is kept (as the hardware cvt and torch do)
    assert orc.encode_e4m3(-1e-6) == 0x80 == int(torch_encode_f32(np.array([-1e-6]))[0])
    assert orc.encode_e4m3(0.0) == 0x00 and orc.encode_e4m3(-0.0) == 0x80
    # R9: satfinite beyond 448 (torch is non-saturating there, so this is a reading, not a pin)
    assert orc.encode_e4m3(1000.0) == 0x7E and orc.encode_e4m3(-1000.0) == 0xFE


def test_encode_invariants(orc):
    # SPEC codec properties: exhaustive round trip, monotone, idempotent grid snap
    t = torch_decode_table()
    for c in range(256):
        if c in (0x7F, 0xFF):
            continue
        assert orc.encode_e4m3(float(t[c])) == c
    rng = np.random.default_rng(1)
    v = np.sort(rng.uniform(-448, 448, 5000))
    dec = [orc.decode_e4m3(orc.encode_e4m3(float(x))) for x in v]
    assert all(a <= b for a, b in zip(dec, dec[1:]))
    for x in v[:500]:
        c = orc.encode_e4m3(float(x))
        assert orc.encode_e4m3(orc.decode_e4m3(c)) == c


# ---------------------------------------------------------------------------------- C3 scale
def _least_T_exact(amax: float) -> int:
    """Independent exact evaluation of 'least integer T with amax <= 448 * 2^T' (Eq. 2 with a
    power-of-two scale rounded up, P:140 + P:173-175) using integer arithmetic only."""
    num, den = amax.as_integer_ratio()                 # amax = num / den exactly
    # guess from bit lengths, then fix up by exact comparison
    T = (num.bit_length() - den.bit_length()) - 9
    def covers(t):                                       # amax <= 448 * 2^t
        return num * (2 ** max(-t, 0)) <= 448 * den * (2 ** max(t, 0))
    while not covers(T):
        T += 1
    while covers(T - 1):
        T -= 1
    return max(-127, min(127, T))


def test_scale_exhaustive_bf16(orc):
    bits = np.arange(0x0001, 0x7F80, dtype=np.uint16)   # every positive finite BF16 incl. subnormals
    vals = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()
    ours = np.array([orc.scale_exponent(float(a)) for a in vals])
    ref = np.array([_least_T_exact(float(a)) for a in vals])
    assert np.array_equal(ours, ref)
    assert ours.min() == -127 and ours.max() == 120     # BF16 range; only the low clamp binds (R13)


def test_scale_examples(orc):
    assert orc.scale_exponent(448.0) == 0               # SPEC tile_quant example (P:143 max)
    assert orc.scale_exponent(600.0) == 1               # SPEC: 600/448 -> 2^1
    assert orc.scale_exponent(1.0) == -8                # 1 <= 448 * 2^-8 = 1.75
    assert orc.scale_exponent(0.0) == -127              # R11: zero tile is neutral


# ---------------------------------------------------------------------------------- C5 shift
def test_shift_bruteforce_all_codes_all_k(orc):
    """shift(c, k) == library RNE cast of decode(c) * 2^-k for all 254 non-NaN codes x k=0..40."""
    t = torch_decode_table()
    codes = [c for c in range(256) if c not in (0x7F, 0xFF)]
    for k in range(41):
        vals = np.array([t[c] * 2.0 ** -k for c in codes], dtype=np.float64)
        assert np.all(vals.astype(np.float32).astype(np.float64) == vals)   # exact in fp32
        ref = torch_encode_f32(vals)
        ours = np.array([orc.shift_e4m3(c, k) for c in codes], dtype=np.uint8)
        assert np.array_equal(ours, ref), k


def test_shift_is_exponent_edit_when_no_underflow(orc):
    """Derivation after Eq. 11: SN' = SN, E' = E - D, M' = M when E - D >= 1."""
    for c in range(256):
        E, M = (c >> 3) & 15, c & 7
        if (E == 15 and M == 7) or E == 0:
            continue
        for k in range(0, E):
            assert orc.shift_e4m3(c, k) == (c & 0x80) | ((E - k) << 3) | M


def test_shift_examples_and_nan(orc):
    with open(os.path.join(GOLDEN, "worked_examples.json")) as f:
        ex = json.load(f)["shift"]
    for e in ex["cases"]:
        assert orc.shift_e4m3(int(e["code"], 16), e["k"]) == int(e["out"], 16), e
    assert orc.shift_e4m3(0x7F, 3) == 0x7F and orc.shift_e4m3(0xFF, 0) == 0xFF
    assert all(orc.shift_e4m3(c, 19) in (0x00, 0x80) for c in range(256) if c not in (0x7F, 0xFF))
    assert orc.shift_e4m3(0x7E, 18) == 0x01             # 448 * 2^-18 = 2^-9.19.. -> 2^-9


# ---------------------------------------------------------------------------------- BF16 round
def test_round_bf16_matches_torch(orc):
    rng = np.random.default_rng(3)
    v = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-30, 30, 20000),
                        (np.arange(1, 2000) * 2.0 ** -16 + 1.0)]).astype(np.float32)
    ref = torch.from_numpy(v).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    ours = np.array([orc.round_bf16(float(x)) for x in v], dtype=np.uint16)
    assert np.array_equal(ours, ref)


def test_checksum_closed_form(orc):
    b = np.array([1, 2, 0, 255], np.uint8)
    phi = 0x9E3779B97F4A7C15
    ref = sum(int(x) * ((i * phi + 1) % 2 ** 64) for i, x in enumerate(b)) % 2 ** 64
    assert orc.checksum64(b) == ref

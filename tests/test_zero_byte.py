"""K1a survivor test (K1a): the per-byte flags of (K - 0x01010101) & ~K & 0x80808080 must
equal "byte is zero" for every code word the scan kernels can produce.  Since r1d the sign-bit gather
leaves copies of the last condition bit in the low bits (2D: bits 3..0 repeat bit 4; 3D: bits 1, 0
repeat bit 2), and ANDs over corners / ORs with AND-neutral bytes keep every low bit <= that bit.  This
checks the claim on all pairs of such bytes (a borrow only travels from a byte to the next one up) and
on random 4-byte words."""
import random

import pytest


def allowed(b: int, lowmask: int, bit: int) -> bool:
    # every low bit set implies the condition bit it repeats is set
    return (b & lowmask) == 0 or bool(b & bit)


def flags(word: int) -> int:
    return ((word - 0x01010101) & ~word & 0x80808080) & 0xFFFFFFFF


@pytest.mark.parametrize("lowmask,bit", [(0x0F, 0x10), (0x03, 0x04)], ids=["2d", "3d"])
def test_zero_byte_flags_exact_on_byte_pairs(lowmask, bit):
    vals = [b for b in range(256) if allowed(b, lowmask, bit)]
    assert 0x01 not in vals and (0x02 not in vals)
    for lo in vals:
        for hi in vals:
            w = lo | (hi << 8) | (0xFF << 16) | (0xFF << 24)
            f = flags(w)
            assert bool(f & 0x80) == (lo == 0)
            assert bool(f & 0x8000) == (hi == 0), (hex(lo), hex(hi))


@pytest.mark.parametrize("lowmask,bit", [(0x0F, 0x10), (0x03, 0x04)], ids=["2d", "3d"])
def test_zero_byte_flags_exact_on_words(lowmask, bit):
    rng = random.Random(7)
    vals = [b for b in range(256) if allowed(b, lowmask, bit)]
    pool = vals + [0] * 64  # zero bytes common, so runs of zeros below nonzero bytes occur
    for _ in range(20000):
        bs = [rng.choice(pool) for _ in range(4)]
        w = bs[0] | bs[1] << 8 | bs[2] << 16 | bs[3] << 24
        f = flags(w)
        for i in range(4):
            assert bool(f >> (8 * i + 7) & 1) == (bs[i] == 0)


def test_plain_formula_is_not_exact_without_the_invariant():
    # the invariant matters: 0x01 above a zero byte is flagged by the borrow
    w = 0x00 | (0x01 << 8) | (0xFF << 16) | (0xFF << 24)
    assert flags(w) & 0x8000

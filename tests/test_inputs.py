"""The seeded input generators (ftk_inputs) -- shared by both sides of every parity test."""
import math

import torch

import ftk_inputs as fi


def test_splitmix64_matches_reference():
    xs = [0, 1, 2, 12345, 2**40 + 7, 2**62 + 3]
    got = fi.splitmix64(torch.tensor(xs, dtype=torch.int64)).tolist()
    for x, g in zip(xs, got):
        assert g & ((1 << 64) - 1) == fi.splitmix64_ref(x)


def test_noise_is_standard_normal():
    z = fi.gaussian_noise(torch.arange(200000, dtype=torch.int64), 0)
    assert abs(float(z.mean())) < 0.01 and abs(float(z.std()) - 1.0) < 0.01


def test_woven_constants():
    w = fi.CONFIGS["C1"].make()
    assert abs(w.dt - 0.02281) < 1e-5  # C1 dt
    w2 = fi.CONFIGS["C2"].make()
    assert abs(w2.h - 15 / 127) < 1e-15 and abs(w2.width - 15 / 127 * 1023) < 1e-12
    f = w.generate(nt=1, dtype=torch.float64)
    X = (torch.arange(32, dtype=torch.float64) / 31 - 0.5) * 15
    assert torch.allclose(f[0, 5], torch.cos(X) * math.sin(X[5].item()))  # t = 0: cos x sin y


def test_moving_extremum_exact_in_fp32():
    me = fi.CONFIGS["C3"].make(nt=3)
    f32 = me.generate(dtype=torch.float32)
    f64 = me.generate(dtype=torch.float64)
    assert torch.equal(f32.double(), f64)
    assert torch.equal(f64 * 256, torch.round(f64 * 256))

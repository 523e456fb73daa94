"""Host side of the counter-based input generator (gen/): recipe statistics and bf16 rounding."""
import numpy as np
import torch

import gen
from gen import CONFIGS


def test_deterministic_and_offsettable():
    a = gen.host_f32(3, gen.X, gen.NORMAL, 1.0, 1000)
    b = gen.host_f32(3, gen.X, gen.NORMAL, 1.0, 400, idx0=600)
    assert np.array_equal(a[600:], b)
    assert not np.array_equal(a, gen.host_f32(4, gen.X, gen.NORMAL, 1.0, 1000))
    assert not np.array_equal(a, gen.host_f32(3, gen.WG, gen.NORMAL, 1.0, 1000))


def test_distributions():
    n = 1 << 20
    x = gen.host_f32(0, gen.X, gen.NORMAL, 1.0, n).astype(np.float64)
    assert abs(x.mean()) < 5e-3 and abs(x.std() - 1) < 5e-3
    assert abs(np.mean(x ** 4) / np.mean(x ** 2) ** 2 - 2.7) < 0.03   # Irwin-Hall(4): excess kurtosis -6/(5*4)
    u = gen.host_f32(0, gen.W1, gen.UNIFORM, 0.25, n).astype(np.float64)
    assert u.min() >= -0.25 and u.max() < 0.25 and abs(u.std() - 0.25 / np.sqrt(3)) < 1e-3
    g = gen.host_f32(0, gen.X, gen.GRID8, 1.0, n)
    assert set(np.unique(g).tolist()) == {q / 8 for q in range(-7, 8)}
    assert (gen.host_f32(0, gen.BG, gen.ZERO, 1.0, 10) == 0).all()


def test_bf16_rounding_matches_torch():
    f = gen.host_f32(1, gen.X, gen.NORMAL, 3.0, 1 << 16)
    f = np.concatenate([f, np.array([0.0, -0.0, 1.0, 1.00390625, 1.0078125, 65504.0, 3.4e38, 1e-40, -1e-40], np.float32)])
    ours = gen.host_bf16_bits(1, gen.X, gen.NORMAL, 3.0, 1 << 16)
    want = torch.from_numpy(f[: 1 << 16].copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, want)
    up = gen.bf16_bits_to_f64(ours)
    assert np.array_equal(up, torch.from_numpy(want.view(np.int16)).view(torch.bfloat16).double().numpy())


def test_masks():
    m = gen.host_mask(0, gen.RESPONDED, 0.3, 100000)
    bits = gen.unpack_mask(m, 100000)
    assert abs(bits.mean() - 0.7) < 0.01
    assert gen.unpack_mask(gen.host_mask(0, gen.ALIVE, 0.0, 77), 77).all()


def test_configs_match_baseline():
    c = CONFIGS
    assert (c["tiny"].E, c["tiny"].D, c["tiny"].H, c["tiny"].k, c["tiny"].T, c["tiny"].dtype) == (16, 64, 256, 4, 32, "f32")
    assert (c["mnist"].E, c["mnist"].D, c["mnist"].k, c["mnist"].T, c["mnist"].fail_frac) == (256, 256, 4, 4096, 0.1)
    assert (c["transformer"].E, c["transformer"].D, c["transformer"].H, c["transformer"].T) == (4096, 1024, 4096, 65536)
    assert (c["grid3d"].E, c["grid3d"].d, c["grid3d"].T) == (4096, 3, 262144)
    assert (c["stress"].E, c["stress"].D, c["stress"].H, c["stress"].k, c["stress"].T, c["stress"].fail_frac) == (4096, 2048, 8192, 8, 1 << 20, 0.3)

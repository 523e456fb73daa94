"""Device side of the generator equals the host side bit for bit (so both halves see one input)."""
import numpy as np
import pytest
import torch

import gen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dist,scale", [(gen.NORMAL, 1.0), (gen.NORMAL, 0.03125), (gen.UNIFORM, 0.0625),
                                        (gen.GRID8, 1.0)])
def test_device_equals_host(dist, scale):
    n = 100003
    for tid in (gen.X, gen.W1):
        d32 = gen.dev_fill(torch.empty(n, dtype=torch.float32, device="cuda"), 5, tid, dist, scale, idx0=77)
        assert np.array_equal(d32.cpu().numpy(), gen.host_f32(5, tid, dist, scale, n, idx0=77))
        dbf = gen.dev_fill(torch.empty(n, dtype=torch.bfloat16, device="cuda"), 5, tid, dist, scale)
        assert np.array_equal(dbf.view(torch.int16).cpu().numpy().view(np.uint16),
                              gen.host_bf16_bits(5, tid, dist, scale, n))
    m = gen.dev_mask(torch.empty(4000, dtype=torch.int32, device="cuda"), 3, gen.RESPONDED, 0.3, 4000 * 32)
    assert np.array_equal(m.cpu().numpy().view(np.uint32), gen.host_mask(3, gen.RESPONDED, 0.3, 4000 * 32))

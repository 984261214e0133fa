"""mpps_level_exps (fp32 Horner level scalings on the device) equals the
host rule engine._exps_for (-round-half-even(log2 norm), 0 for zero or
non-finite norms) on every level selected by the mask."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_level_exps_matches_host_rule(cuda):
    import torch
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.engine import _exps_for
    rng = np.random.default_rng(0)
    B, r = 37, 6
    norms = 10.0 ** rng.uniform(-300, 300, (B, r + 2))
    norms[3, 2] = 0.0
    norms[4, 5] = np.inf
    norms[5, 1] = np.nan
    norms[6, :] = 2.0 ** np.arange(-3, r - 1) * 1.5        # ties of log2 -> half-even
    mask = (1 << 2) | (1 << 4) | (1 << 5)
    h = _lib.handle_for()
    nd = torch.from_numpy(norms).to(cuda)
    exps = torch.empty((r + 2, B), dtype=torch.int32, device=cuda)
    ey = torch.empty((B,), dtype=torch.int32, device=cuda)
    h.level_exps(nd, r, mask, exps, ey)
    want = _exps_for(norms)                                   # (B, r+2)
    got = exps.cpu().numpy()
    for j in range(r + 2):
        if (mask >> j) & 1:
            assert np.array_equal(got[j], want[:, j]), j
        else:
            assert not got[j].any(), j
    assert np.array_equal(ey.cpu().numpy(), want[:, r + 1])

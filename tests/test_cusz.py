"""cuSZ dual quantization -> GPULZ on the device (the paper's use case,
PAPER.md Table 3).  The quantizer and its inverse are
checked bit-exactly against the numpy restatement oracle/cusz_oracle.py, the
error bound |f - f'| <= eb is checked on the reconstruction, and the whole
field -> codes -> GPULZ image -> field path round-trips."""
import numpy as np
import pytest

import cusz_oracle as Q


def smooth_field(shape, seed, spikes=0):
    rs = np.random.default_rng(seed)
    grids = np.meshgrid(*[np.linspace(0, 1, n, dtype=np.float64) for n in shape], indexing="ij")
    f = np.zeros(shape)
    for _ in range(6):
        term = rs.random() * 3
        for g in grids:
            term = term * np.sin(g * rs.random() * 12 + rs.random() * 6)
        f += term
    f += 0.002 * rs.standard_normal(shape)
    if spikes:
        flat = f.reshape(-1)
        flat[rs.integers(0, flat.size, spikes)] += rs.normal(0, 50, spikes)
    return f.astype(np.float32)


def test_oracle_round_trip_and_error_bound():
    for shape in [(37,), (19, 23), (7, 11, 13)]:
        f = smooth_field(shape, 1, spikes=5)
        eb = 1e-3 * float(f.max() - f.min())
        codes, idx, val = Q.lorenzo_quantize(f, eb, 64)
        dims = (1,) * (3 - len(shape)) + shape
        back = Q.lorenzo_reconstruct(codes, idx, val, dims, eb, 64).reshape(shape)
        assert np.abs(back - f).max() <= eb * (1 + 1e-4) + 1e-6
        assert len(idx) >= 1  # the spikes are outliers


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1000,), (64, 77), (9, 40, 33), (26, 180, 360)])
@pytest.mark.parametrize("radius", [512, 8])
def test_quantize_matches_oracle(shape, radius):
    import torch

    from paper_2304_07342_b200 import cusz

    f = smooth_field(shape, sum(shape), spikes=3)
    eb = 1e-3 * float(f.max() - f.min())
    q = cusz.quantize(torch.from_numpy(f).cuda(), eb, radius)
    codes, idx, val = Q.lorenzo_quantize(f, eb, radius)
    assert np.array_equal(q.codes.cpu().numpy().view(np.uint16), codes)
    assert np.array_equal(q.outlier_idx.cpu().numpy(), idx)
    assert np.array_equal(q.outlier_val.cpu().numpy(), val)
    back = cusz.reconstruct(q).cpu().numpy().reshape(shape)
    dims = (1,) * (3 - len(shape)) + shape
    want = Q.lorenzo_reconstruct(codes, idx, val, dims, eb, radius).reshape(shape)
    assert np.array_equal(back, want)
    assert np.abs(back - f).max() <= eb * (1 + 1e-4) + 1e-6


@pytest.mark.gpu
def test_field_through_gpulz_round_trip():
    import torch

    from paper_2304_07342_b200 import cusz, plz

    f = smooth_field((26, 180, 360), 3, spikes=20)
    eb = 1e-3 * float(f.max() - f.min())
    d = torch.from_numpy(f).cuda()
    for I in (1, 2):
        cf = cusz.compress_field(d, eb, plz.validate(plz.Params(2, 255, 2048, I)))
        assert cf.image.is_cuda
        q = cusz.quantize(d, eb)
        assert bytes(plz.decompress_bytes(cf.image).cpu().numpy().tobytes()) == \
            bytes(q.codes.cpu().numpy().tobytes())
        back = cusz.decompress_field(cf)
        assert float((back - d).abs().max()) <= eb * (1 + 1e-4) + 1e-6
        assert f.nbytes / cf.nbytes > 4.0  # codes of a smooth field compress well


@pytest.mark.gpu
def test_quantize_rejects_bad_arguments():
    import torch

    from paper_2304_07342_b200 import cusz, plz

    with pytest.raises(plz.ValidationError):
        cusz.quantize(torch.zeros(10, device="cuda"), 0.0)
    with pytest.raises(plz.ValidationError):
        cusz.quantize(torch.zeros(10, device="cuda"), 1e-3, radius=40000)
    with pytest.raises(plz.ValidationError):
        cusz.quantize(torch.zeros(10), 1e-3)

""".spkb straight into HBM and back (spk_spkb_load / spk_spkb_store, SURVEY.md
section 8(f) row 3), against the reference-written fixtures and the host path."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
SEED = 20181108


def test_device_load_and_store_reference_file(oracle, spk, tmp_path):
    path = os.path.join(GOLD, "ref_n257_kl16_ku2.spkb")
    n, kl, ku = spk.spkb_header(path)
    d = torch.empty((n, kl + ku + 1), dtype=torch.float64, device="cuda")
    spk.load_spkb_device(path, d.data_ptr())
    assert np.array_equal(d.cpu().numpy(), oracle.generate_band(SEED + n, n, kl, ku, 1.2))
    out = tmp_path / "back.spkb"
    spk.store_spkb_device(out, d.data_ptr(), n, kl, ku)
    assert out.read_bytes() == open(path, "rb").read()


def test_multichunk_round_trip_and_slab_windows(oracle, spk, tmp_path):
    """A file larger than the 64 MB staging chunk; slab windows with halos."""
    from paper_1811_03559_b200 import distributed as D

    n, k = 70000, 64
    dev = torch.device("cuda", 0)
    band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
    spk.generate_band_device(5, n, k, k, 1.3, band.data_ptr())
    torch.cuda.synchronize()
    path = tmp_path / "big.spkb"
    spk.store_spkb_device(path, band.data_ptr(), n, k, k)
    assert os.path.getsize(path) == 28 + 8 * n * (2 * k + 1)
    back = torch.full_like(band, float("nan"))
    spk.load_spkb_device(path, back.data_ptr())
    assert torch.equal(back, band)
    host = spk.read_spkb(path)
    assert np.array_equal(host.data, band.cpu().numpy())
    for G in (2, 3):
        rows = D.slab_rows(n, G)
        for g in range(G):
            t, shape, lh = D.load_slab_band(path, g, G)
            assert shape == (n, k, k)
            _, rh = D.halo(g, G, k)
            assert torch.equal(t, band[rows[g] - lh:rows[g + 1] + rh])


def test_factorize_from_loaded_band(oracle, spk, tmp_path):
    """A band loaded from .spkb solves like the in-memory one (same bits in)."""
    path = os.path.join(GOLD, "ref_n300_kl3_ku5.spkb")
    a = spk.read_spkb(path)
    F = np.asfortranarray(oracle.generate_rhs(7, a.n, 2))
    fact = spk.factorize(a, spk.gpu_plan(a.n, a.kl, a.ku, 2, False, 3))
    X = spk.solve(fact, F)
    assert spk.relative_residual(a, X, F) <= 1e-12

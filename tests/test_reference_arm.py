"""The bench's reference arm (bench.py --impl reference): the UNMODIFIED reference run_lp
(oracle/_ref) with the fp32 CPU DiT (oracle/cpu_dit.py) in its Denoiser slot.  CPU-only,
at toy sizes, so the round-end reference run cannot fail on plumbing."""
import numpy as np
import pytest

from oracle.cpu_dit import CpuDiT, dit_flops

SMALL = dict(dim=256, num_heads=2, ffn_dim=512, text_len=16, text_dim=64, freq_dim=32)


def test_cpu_dit_predict_shapes_and_cfg_passes():
    dit = CpuDiT(num_layers=1, **SMALL)
    z = np.random.default_rng(0).standard_normal((16, 3, 6, 8))
    u = dit.predict(z, 4, np.zeros(0), True)
    c = dit.predict(z, 4, np.ones(8), False)
    assert u.shape == z.shape and c.shape == z.shape
    assert np.isfinite(u).all() and np.isfinite(c).all()
    assert not np.allclose(u, c)        # uncond (null text) and cond passes differ
    assert len(dit.calls) == 2


def test_reference_run_lp_with_cpu_dit(reference):
    dit = CpuDiT(num_layers=1, **SMALL)
    z, cond = reference.synthetic((16, 4, 8, 8), 4, 2025)
    out, ledger = reference.run_lp_callback(dit.predict, z, 4, 2, 0.05, 5.0, cond, (1, 2, 2), 2, 0.5)
    assert out.shape == z.shape and np.isfinite(out).all() and ledger > 0
    assert len(dit.calls) == 2 * 2 * 2      # steps x workers x CFG passes


def test_dit_flops_matches_bench_formula():
    # one block, one CFG pass on a 1x2x2-patch shard: GEMMs 2n(6d^2+2dF) + self 4n^2 d + cross 4n*512*d
    n = 21 * 30 * 52
    want = 2 * n * (6 * 1536 ** 2 + 2 * 1536 * 8960) + 4 * n * n * 1536 + 4 * n * 512 * 1536
    assert dit_flops((16, 21, 60, 104), (1, 2, 2)) == want


@pytest.mark.parametrize("shape", [(16, 9, 60, 104)])
def test_bench_reference_flop_scale_is_cycle_over_t_axis(reference, shape):
    from oracle.oracle import sub_shape

    def axis(step):
        p = reference.build_plan((16, 21, 60, 104), (1, 2, 2), step, 4, 0.5)
        return sum(dit_flops(sub_shape((16, 21, 60, 104), p, k), (1, 2, 2)) for k in range(p.n))

    scale = 30 * sum(axis(s) for s in (1, 2, 3)) / 3 / axis(1)
    assert 25 < scale < 30   # the T axis is the most expensive of the cycle

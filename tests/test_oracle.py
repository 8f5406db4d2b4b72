"""Pin the oracle before trusting it: the numpy and C restatements of the reference ring
reproduce, bit for bit, the outputs of the reference's real multi-process TCP ring
(tests/golden/ring.npz, made by tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import golden_ring
from oracle import ring_oracle

RING_N = (2, 3, 4, 8)
RING_SIZES = (1, 17, 1001, 4099)


def _inputs(n_ranks, n):
    g = golden_ring()
    return [g[f"in_N{n_ranks}_n{n}_r{r}"] for r in range(n_ranks)], g[f"out_N{n_ranks}_n{n}"]


def test_segments_match_reference_rules():
    assert ring_oracle.segments(10, 4) == ([3, 3, 2, 2], [0, 3, 6, 8])
    assert ring_oracle.segments(1, 8)[0] == [1, 0, 0, 0, 0, 0, 0, 0]
    assert ring_oracle.segments(0, 3) == ([0, 0, 0], [0, 0, 0])


@pytest.mark.parametrize("n_ranks", RING_N)
@pytest.mark.parametrize("n", RING_SIZES)
def test_numpy_ring_matches_reference_bits(n_ranks, n):
    ins, want = _inputs(n_ranks, n)
    for out in ring_oracle.ring_allreduce_numpy(ins):
        assert np.array_equal(out.view("<u4"), want.view("<u4"))


@pytest.mark.parametrize("n_ranks", RING_N)
@pytest.mark.parametrize("n", RING_SIZES)
@pytest.mark.parametrize("threads", [1, None])
def test_c_ring_matches_reference_bits(n_ranks, n, threads):
    if not ring_oracle.have_c():
        pytest.skip("C oracle not built (make -C oracle)")
    ins, want = _inputs(n_ranks, n)
    for out in ring_oracle.ring_allreduce_c(ins, threads=threads):
        assert np.array_equal(out.view("<u4"), want.view("<u4"))


def test_fold_order_is_load_bearing():
    """A naive rank-0-first sum differs from the reference bits on random data,
    so matching the golden outputs really pins the fold order."""
    ins, want = _inputs(8, 4099)
    naive = ins[0].copy()
    for x in ins[1:]:
        naive = naive + x
    assert not np.array_equal(naive.view("<u4"), want.view("<u4"))


def test_segment_rotated_left_fold_equals_ring():
    ins, want = _inputs(4, 1001)
    sizes, offsets = ring_oracle.segments(1001, 4)
    out = np.empty(1001, dtype="<f4")
    for s in range(4):
        sl = slice(offsets[s], offsets[s] + sizes[s])
        acc = ins[s][sl].copy()
        for k in range(1, 4):
            acc = acc + ins[(s + k) % 4][sl]
        out[sl] = acc
    assert np.array_equal(out.view("<u4"), want.view("<u4"))


def test_pack_layout_high_layer_first():
    counts = [5, 0, 7, 3]
    vals = {1: np.full(5, 1, "<f4"), 3: np.full(7, 3, "<f4"), 4: np.full(3, 4, "<f4")}
    bucket = ring_oracle.pack_group(vals, counts, 1, 4)
    assert bucket.tolist() == [4.0] * 3 + [3.0] * 7 + [1.0] * 5
    back = ring_oracle.unpack_group(bucket, counts, 1, 4)
    assert set(back) == {1, 3, 4} and all(np.array_equal(back[k], vals[k]) for k in back)
    assert ring_oracle.emulation_expected(4, 7) == 10 + 4 * 2


def test_bf16_rounding_matches_torch_cast():
    import torch

    from oracle import ring_oracle

    rng = np.random.default_rng(5)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 20000),
                        np.array([0.0, -0.0, 1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, 3.3895314e38, 1e-40, -1e-40],
                                 dtype=np.float32)]).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ring_oracle.bf16_round(x), want)
    assert np.array_equal(ring_oracle.bf16_to_f32(want), torch.from_numpy(want.view(np.int16)).view(torch.bfloat16).float().numpy())


def test_bf16_ring_is_fp32_fold_rounded_once():
    from oracle import ring_oracle

    rng = np.random.default_rng(9)
    for n_ranks in (2, 3, 8):
        ins = [ring_oracle.bf16_round(rng.standard_normal(1001).astype(np.float32)) for _ in range(n_ranks)]
        got = ring_oracle.ring_allreduce_bf16(ins)
        folded = ring_oracle.ring_allreduce([ring_oracle.bf16_to_f32(v) for v in ins])[0]
        assert np.array_equal(got, ring_oracle.bf16_round(folded))
        # integers are exact in both formats: the reference's exact-sum pattern survives
        ones = [ring_oracle.bf16_round(np.full(17, r + 1, np.float32)) for r in range(n_ranks)]
        assert np.all(ring_oracle.bf16_to_f32(ring_oracle.ring_allreduce_bf16(ones)) == n_ranks * (n_ranks + 1) / 2)
        half = ring_oracle.ring_allreduce_bf16(ones, scale=0.5)
        assert np.all(ring_oracle.bf16_to_f32(half) == n_ranks * (n_ranks + 1) / 4)

"""Maximum sizes: one shard of more than 2^31 codes on one GPU (the scan runs in 2^30-code
windows; histogram counts are uint32; repair keys carry 32-bit code indices).  One Lloyd
iteration through the ShardEngine with two clusters forced empty (duplicate centers lose
every tie to the lower index), checked on sampled rows against the oracle's exact scan
(including rows at both sides of 2^31), on the histogram totals, on the objective against
an independent float64 sum, and on the repair choice (largest sd, lowest index first)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_shard_above_2_31_codes(oracle):
    import torch

    from paper_1709_03708_b200 import _lib, engine

    n = (1 << 31) + 12345
    m, l, k = 4, 256, 8
    rng = np.random.default_rng(0)
    tables = oracle.build_distance_tables(rng.normal(size=(m, l, 2)).astype(np.float32))
    dev = engine.device_of()
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    codes_dev = torch.randint(0, 256, (n, m), generator=g, device=dev, dtype=torch.uint8)
    centers = rng.integers(0, 256, size=(k, m)).astype(np.uint8)
    centers[6] = centers[0]
    centers[7] = centers[0]
    eng = engine.ShardEngine(codes_dev, engine.device_tables(tables, dev), k, dev)
    eng.assign(engine.upload_codes(centers, m, dev))
    eng.objective()
    eng.histogram()
    eng.vote()
    sums, stats = eng.read_obj_stats()
    assert stats[_lib.STAT_EMPTY] == 2 and stats[_lib.STAT_FILLED] == k - 2
    eng.repair()

    idx = np.concatenate([rng.integers(0, n, size=3000), np.arange(n - 40, n), np.arange(0, 40),
                          np.arange((1 << 31) - 20, (1 << 31) + 20), np.arange((1 << 30) - 20, (1 << 30) + 20)])
    sel = torch.from_numpy(idx).to(dev)
    codes_s = codes_dev[sel].cpu().numpy()
    ref_lab, ref_sd = oracle.assign_c(codes_s, centers, tables, threads=4, want_sd=True)
    np.testing.assert_array_equal(eng.labels[sel].cpu().numpy().view(np.uint32), ref_lab.astype(np.uint32))
    np.testing.assert_array_equal(eng.sd[sel].cpu().numpy(), ref_sd)

    sd = eng.sd[:n]
    total = float(sd.sum().item())
    assert abs(sums[1] - total) <= 1e-9 * abs(total)
    cnt = eng.counts.cpu().numpy().view(np.uint32).astype(np.int64)
    assert cnt.sum() == n and cnt[6] == 0 and cnt[7] == 0
    hist = eng.hist.view(k, m, l).cpu().numpy().view(np.uint32).astype(np.int64)
    np.testing.assert_array_equal(hist.sum(axis=2), np.repeat(cnt[:, None], m, axis=1))

    # repair: clusters 6, 7 take the codes with the largest sd, lowest index first
    v1 = sd.max()
    at1 = torch.nonzero(sd == v1).flatten()
    i1 = int(at1[0])
    if at1.numel() > 1:
        i2 = int(at1[1])
    else:
        v2 = sd[sd < v1].max()
        i2 = int(torch.nonzero(sd == v2).flatten()[0])
    newc = eng.new_centers[:, :m].cpu().numpy()
    np.testing.assert_array_equal(newc[6], codes_dev[i1].cpu().numpy())
    np.testing.assert_array_equal(newc[7], codes_dev[i2].cpu().numpy())

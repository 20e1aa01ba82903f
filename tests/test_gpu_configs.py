"""Parity at the BASELINE.json configurations, on the default path (8-bit first tier at
M = 4: configs 2 and 4; 16-bit at M = 8 / 16: configs 3 and 5; fp32 scan for config 1).

Each workload is built exactly as bench.py builds it (bench.build_workload: the
reference-trained codebook of bench_assets/, the same seeded vectors, the GPU
encoder), then Lloyd iterations run through the same engine the bench times
(eager first iteration, CUDA-graph replay afterwards) and every iteration's state is
checked against the oracle by bench.parity_record:

- labels and sd_sq of sampled codes, bit for bit (clustering.py:167-197, pq.py:271-290;
  oracle.assign_c, the C restatement pinned to the reference in test_oracle_golden);
- the objective sums (numpy's pairwise tree, clustering.py:448-449);
- the full K x M x 256 histogram and the counts (clustering.py:344-347, :458);
- sampled (k, m) votes (clustering.py:349-354, exact-arithmetic argmin);
- every repaired cluster (clustering.py:460-466).

Config 2 additionally runs a 3-iteration fit against the oracle's fit on all 1e6
codes.  Configs 4 and 5 are the per-GPU shards of the 8-GPU runs at full size.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _engine_iterations(cfg_name, iterations, rows, votes=2000, n_loc=None):
    import torch

    import bench
    from paper_1709_03708_b200 import _lib, engine

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = bench.CONFIGS[cfg_name]
    wl = bench.build_workload(cfg_name, dev, n_loc=n_loc)
    codes_host, tables = wl["codes_host"], wl["tables"]
    n, k, m, l_count = wl["n_loc"], cfg["k"], cfg["m"], cfg["l"]
    with torch.cuda.device(dev):
        dt = engine.device_tables(tables, dev)
        eng = engine.ShardEngine(engine.upload_codes(codes_host, m, dev), dt, k, dev)
        cur = engine.upload_codes(codes_host[bench.center_indices(n, k)], m, dev)
        graphs = None
        records = []
        for it in range(iterations):
            cur_in = cur.clone()
            if graphs is None:
                eng.assign(cur)
                eng.objective()
                eng.histogram()
                eng.vote()
                _, st = eng.read_obj_stats()
                if st[_lib.STAT_EMPTY]:
                    eng.repair()
                cur = eng.new_centers.clone()
                graphs = engine.IterationGraphs(eng, cur)
            else:
                graphs.main.replay()
                _, st = eng.read_obj_stats()
                if st[_lib.STAT_EMPTY]:
                    graphs.repair.replay()
                cur.copy_(eng.new_centers)
            torch.cuda.synchronize(dev)
            rec = bench.parity_record(eng, cur_in, codes_host, tables, k, m, l_count, rows=rows, votes=votes,
                                      seed=1000 + it)
            rec["lookup_bytes"] = int(st[_lib.STAT_LOOKUP_BYTES])
            rec["flagged"] = int(st[_lib.STAT_FLAGGED])
            records.append(rec)
    return wl, records


def _assert_clean(records, first_tier_bytes):
    for i, rec in enumerate(records):
        assert rec["mismatch"] == 0, (i, rec)
        assert rec["objective_equal"], (i, rec)
        assert rec["lookup_bytes"] == first_tier_bytes, (i, rec)  # the default first tier ran


def test_config2_full_rows():
    """Config 2 (N=1e6, K=1e4, M=4): every code's label and sd, two iterations."""
    _, recs = _engine_iterations("c2", 2, rows=1_000_000)
    _assert_clean(recs, first_tier_bytes=1)
    assert recs[0]["rows"] == 1_000_000


def test_config2_fit_vs_oracle(oracle):
    """Three iterations of fit (eager + graph replay) against the oracle's fit with the C scan."""
    import torch

    import bench
    import paper_1709_03708_b200 as pqk

    dev = torch.device("cuda", 0)
    wl = bench.build_workload("c2", dev)
    codes, tables = wl["codes_host"], wl["tables"]
    k = bench.CONFIGS["c2"]["k"]
    init = codes[bench.center_indices(len(codes), k)]
    res = pqk.fit(codes, tables, k, max_iterations=3, initial_centers=init)
    ref = oracle.fit(codes, tables, k, max_iterations=3, initial_centers=init,
                     scan=lambda c, ce, t: oracle.assign_c(c, ce, t))
    np.testing.assert_array_equal(res.labels, ref["labels"])
    np.testing.assert_array_equal(res.centers, ref["centers"])
    assert [s.objective for s in res.trace] == [t["objective"] for t in ref["trace"]]
    assert [s.objective_sq for s in res.trace] == [t["objective_sq"] for t in ref["trace"]]
    assert [s.repaired_clusters for s in res.trace] == [t["repaired"] for t in ref["trace"]]


def test_config4_shard():
    """Config 4's per-GPU shard (N=1.25e8 SIFT-like codes, K=1e5, M=4): 3,125 chunks of
    32 centres in the 8-bit tier, the fp32 list tier (~6e4 flagged codes per iteration) and
    scan windows of 2^28 codes on the default path."""
    _, recs = _engine_iterations("c4", 2, rows=50_000)
    _assert_clean(recs, first_tier_bytes=1)
    assert recs[0]["hist_bins"] == 100_000 * 4 * 256


def test_config4_encode_sample(oracle):
    """Config 4 codes of the first device-generated chunk against the oracle's encoder."""
    import torch

    import bench
    from paper_1709_03708_b200 import engine

    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS["c4"]
    book = bench.make_codebook("c4", 4, 256)
    s, e, seed = bench.gpu_chunks(cfg, cfg["n"], 0)[0]
    vec = bench.sift_like_gpu(e - s, seed, dev)
    cw = torch.from_numpy(np.array(book)).to(dev)
    codes = engine.encode_device(vec, cw, 4, 256, dev).cpu().numpy()
    rows = np.sort(np.random.default_rng(4).choice(e - s, size=20_000, replace=False))
    x = vec[torch.from_numpy(rows).to(dev)].cpu().numpy()
    np.testing.assert_array_equal(codes[rows], oracle.encode(book, x))


def test_config5_shard():
    """Config 5's per-GPU shard (N=1.25e7 mixture codes, K=1e5, M=16)."""
    _, recs = _engine_iterations("c5", 2, rows=20_000)
    _assert_clean(recs, first_tier_bytes=2)


def test_config3_sampled():
    """Config 3 (N=1e7 deep-feature-like 4096-D vectors encoded by the K-streamed
    tensor-core encoder, K=1e4, M=8)."""
    _, recs = _engine_iterations("c3", 2, rows=50_000)
    _assert_clean(recs, first_tier_bytes=2)


def test_config1_full():
    """Config 1 (N=1e5, K=1e3): below 2^31 lookups the fp32 scan is the first tier."""
    _, recs = _engine_iterations("c1", 3, rows=100_000)
    _assert_clean(recs, first_tier_bytes=4)

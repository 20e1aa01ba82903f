"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Every array is an input or an output of a reference
call (pqclust.assign / fit / encode / update_center_* / build_distance_tables /
paired_distance_sq), or numpy's own np.mean for the objective tree.  The cases
follow the reference tests' scenarios (tests/test_clustering.py, test_pq.py,
test_acceptance.py C1/C4) plus config 1 of BASELINE.json at full size.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parents[1]))

import pqclust  # noqa: E402  (the reference, from /root/reference/pkg/src)
from pqclust import (  # noqa: E402
    PQCodebook,
    assign,
    build_distance_tables,
    build_histogram,
    encode,
    fit,
    paired_distance_sq,
    train_codebook,
    update_center_naive,
    update_center_sparse,
)

assert "/root/reference" in pqclust.__file__, pqclust.__file__


def random_tables(m, l_count, seed=0, sub_dim=2):
    rng = np.random.default_rng(seed)
    book = PQCodebook(rng.standard_normal((m, l_count, sub_dim)).astype(np.float32))
    t = build_distance_tables(book)
    object.__setattr__(t, "_book", book.codewords)
    return t


def lattice_tables(m, l_count):
    grid = np.arange(l_count, dtype=np.float32).reshape(l_count, 1)
    book = PQCodebook(np.broadcast_to(grid, (m, l_count, 1)).copy())
    t = build_distance_tables(book)
    object.__setattr__(t, "_book", book.codewords)
    return t


def tables_record(prefix, t):
    """Tables are stored as their codebook + SHA-256 of the reference's float64
    tables; the tests rebuild them (oracle.build_distance_tables) and check the hash."""
    return {f"{prefix}codebook": t._book, f"{prefix}tables_sha256": np.array(hashlib.sha256(t.tables.tobytes()).hexdigest())}


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(name, sum(a.nbytes for a in arrays.values() if hasattr(a, "nbytes")), "bytes raw")


def pack_fit(prefix, res):
    tr = res.trace
    return {
        f"{prefix}labels": res.labels,
        f"{prefix}centers": res.centers,
        f"{prefix}objective": np.array([s.objective for s in tr]),
        f"{prefix}objective_sq": np.array([s.objective_sq for s in tr]),
        f"{prefix}repaired": np.array([s.repaired_clusters for s in tr]),
        f"{prefix}nnz": np.array([np.nan if s.mean_histogram_nnz is None else s.mean_histogram_nnz for s in tr]),
        f"{prefix}update_zero": np.array([s.update_seconds == 0.0 for s in tr]),
        f"{prefix}iterations_run": np.array(res.iterations_run),
        f"{prefix}converged": np.array(res.converged),
    }


def make_assign():
    arrays = {}
    cases = []
    rng = np.random.default_rng(1234)
    for i, (m, l_count) in enumerate([(1, 16), (2, 64), (3, 16), (4, 256), (5, 32), (8, 256), (16, 256)]):
        t = random_tables(m, l_count, seed=50 + i, sub_dim=3)
        codes = rng.integers(0, l_count, size=(1500, m)).astype(np.uint8)
        centers = rng.integers(0, l_count, size=(77, m)).astype(np.uint8)
        centers[10] = centers[3]
        cases.append((t, codes, centers))
    for i in range(6):  # acceptance C4 lattice + duplicated center rows
        m = [1, 2, 1, 2, 4, 4][i]
        t = lattice_tables(m, 16)
        codes = rng.integers(0, 16, size=(500, m)).astype(np.uint8)
        centers = rng.integers(0, 16, size=(20, m)).astype(np.uint8)
        centers[5] = centers[2]
        cases.append((t, codes, centers))
    # hand tie cases (test_clustering.py:135-143)
    lt = lattice_tables(1, 8)
    for cs in ([[2], [4]], [[4], [2]], [[5], [5], [2]], [[5], [5]]):
        cases.append((lt, np.array([[3]], dtype=np.uint8), np.array(cs, dtype=np.uint8)))
    for i, (t, codes, centers) in enumerate(cases):
        labels = assign(codes, centers, t)
        sd = paired_distance_sq(t, codes, centers[labels])
        arrays.update(tables_record(f"c{i}_", t))
        arrays.update({f"c{i}_codes": codes, f"c{i}_centers": centers,
                       f"c{i}_labels": labels, f"c{i}_sd": sd})
    arrays["ncases"] = np.array(len(cases))
    save("assign", **arrays)


def make_fit():
    arrays = {}
    specs = []
    rng = np.random.default_rng(30)
    for trial in range(10):
        m = int(rng.choice([1, 2, 3, 4, 8]))
        l_count = int(rng.choice([8, 32, 256]))
        t = random_tables(m, l_count, seed=100 + trial)
        n = int(rng.integers(200, 4000))
        codes = rng.integers(0, l_count, size=(n, m)).astype(np.uint8)
        k = int(rng.integers(2, 40))
        specs.append(dict(t=t, codes=codes, k=k, seed=trial, it=15, update="sparse", init=None))
    # clustered codes with many empty clusters (config-1-like repair pressure)
    protos = rng.integers(0, 256, size=(60, 4))
    lab = rng.integers(0, 60, size=8000)
    codes = protos[lab].copy()
    flip = rng.random(codes.shape) < 0.15
    codes[flip] = rng.integers(0, 256, size=int(flip.sum()))
    specs.append(dict(t=random_tables(4, 256, seed=7, sub_dim=8), codes=codes.astype(np.uint8), k=200, seed=3, it=8,
                      update="sparse", init=None))
    # known answers (test_clustering.py:233-305)
    lt = lattice_tables(2, 32)
    kn = np.unique(np.random.default_rng(20).integers(0, 32, size=(64, 2), dtype=np.uint8), axis=0)
    specs.append(dict(t=lt, codes=kn, k=len(kn), seed=0, it=20, update="sparse", init=None))
    specs.append(dict(t=lattice_tables(1, 200), codes=np.array([0, 1, 2, 99, 100, 101, 197, 198, 199], np.uint8)[:, None],
                      k=3, seed=0, it=20, update="sparse", init=np.array([[1], [100], [198]], np.uint8)))
    specs.append(dict(t=lattice_tables(1, 6), codes=np.array([[0], [0], [5], [5]], np.uint8), k=2, seed=0, it=20,
                      update="sparse", init=np.array([[0], [0]], np.uint8)))
    sn_codes = np.random.default_rng(31).integers(0, 64, size=(3000, 4), dtype=np.uint8)
    for upd in ("sparse", "naive"):
        specs.append(dict(t=random_tables(4, 64, seed=32), codes=sn_codes, k=12, seed=5, it=20, update=upd, init=None))
    for i, s in enumerate(specs):
        res = fit(s["codes"], s["t"], s["k"], max_iterations=s["it"], seed=s["seed"], update=s["update"],
                  initial_centers=s["init"])
        arrays.update(tables_record(f"f{i}_", s["t"]))
        arrays.update({f"f{i}_codes": s["codes"], f"f{i}_k": np.array(s["k"]),
                       f"f{i}_seed": np.array(s["seed"]), f"f{i}_it": np.array(s["it"]),
                       f"f{i}_update": np.array(s["update"]),
                       f"f{i}_init": s["init"] if s["init"] is not None else np.zeros((0, 0), np.uint8)})
        arrays.update(pack_fit(f"f{i}_", res))
    arrays["ncases"] = np.array(len(specs))
    save("fit", **arrays)


def make_config1():
    """BASELINE.json configs[0] at full size, every stage by the reference."""
    seed = 1234
    rng = np.random.default_rng(seed)
    means = rng.uniform(0.0, 100.0, size=(1000, 128))
    lab = rng.integers(0, 1000, size=100_000)
    vectors = (means[lab] + rng.normal(0.0, 5.0, size=(100_000, 128))).astype(np.float32)
    sample = vectors[np.random.default_rng(seed + 1).choice(100_000, 20_000, replace=False)]
    book = train_codebook(sample, 4, 256, iterations=20, seed=1)
    codes = encode(book, vectors)
    tables = build_distance_tables(book)
    res = fit(codes, tables, 1000, max_iterations=10, seed=7, threads=8)
    sha = hashlib.sha256(tables.tables.tobytes()).hexdigest()
    save("config1", codebook=book.codewords, codes=codes, tables_sha256=np.array(sha),
         vectors_head=vectors[:512], codes_head=codes[:512], **pack_fit("", res))


def make_encode():
    arrays = {}
    rng = np.random.default_rng(6)
    specs = [(3, 12, 4), (4, 256, 32), (8, 256, 16), (2, 64, 64), (1, 256, 3)]
    for i, (m, l_count, sub) in enumerate(specs):
        book = PQCodebook(np.random.default_rng(5 + i).standard_normal((m, l_count, sub)).astype(np.float32))
        vectors = rng.normal(size=(400, m * sub)).astype(np.float32)
        vectors[:8] = np.concatenate([book.codewords[mm][rng.integers(0, l_count, 8)] for mm in range(m)], axis=1)
        arrays.update({f"e{i}_codewords": book.codewords, f"e{i}_vectors": vectors, f"e{i}_codes": encode(book, vectors)})
    # ties toward low index (test_pq.py:118-125)
    dup = PQCodebook(np.array([[[0.0], [3.0], [3.0], [7.0]]], dtype=np.float32))
    arrays.update({"t0_codewords": dup.codewords, "t0_vectors": np.array([[3.0]], np.float32),
                   "t0_codes": encode(dup, np.array([[3.0]], np.float32))})
    lat = PQCodebook(np.arange(4, dtype=np.float32).reshape(1, 4, 1))
    arrays.update({"t1_codewords": lat.codewords, "t1_vectors": np.array([[0.5]], np.float32),
                   "t1_codes": encode(lat, np.array([[0.5]], np.float32))})
    arrays["ncases"] = np.array(len(specs))
    save("encode", **arrays)


def make_vote():
    """Acceptance C1-style clusters: update_center_sparse == update_center_naive."""
    rng = np.random.default_rng(101)
    arrays = {}
    i = 0
    for m, l_count in [(1, 4), (2, 16), (4, 64), (8, 256), (4, 256)]:
        t = random_tables(m, l_count, seed=9 + m + l_count)
        arrays.update(tables_record(f"t{m}_{l_count}_", t))
        for rep in range(30):
            size = int(rng.integers(1, 1001))
            members = rng.integers(0, l_count, size=(size, m)).astype(np.uint8)
            hists = [build_histogram(members[:, mm], l_count) for mm in range(m)]
            sparse = update_center_sparse(hists, t)
            naive = update_center_naive(members, t)
            assert np.array_equal(sparse, naive)
            arrays[f"v{i}_members"] = members
            arrays[f"v{i}_key"] = np.array(f"t{m}_{l_count}")
            arrays[f"v{i}_center"] = sparse
            i += 1
    # lattice tables: exact ties in the votes (symmetric histograms)
    lt = lattice_tables(1, 16)
    arrays.update(tables_record("lat_", lt))
    for members in ([[3], [5]], [[0], [2], [2], [0]], [[1], [1], [7], [7], [4]]):
        mem = np.array(members, np.uint8)
        arrays[f"v{i}_members"] = mem
        arrays[f"v{i}_key"] = np.array("lat")
        arrays[f"v{i}_center"] = update_center_sparse([build_histogram(mem[:, 0], 16)], lt)
        i += 1
    arrays["ncases"] = np.array(i)
    save("vote", **arrays)


def make_tables_and_mean():
    arrays = {}
    for i, (m, l_count, sub) in enumerate([(4, 256, 32), (8, 256, 16), (2, 16, 3), (16, 256, 8)]):
        book = PQCodebook(np.random.default_rng(70 + i).normal(size=(m, l_count, sub)).astype(np.float32) * 10)
        arrays[f"b{i}_codewords"] = book.codewords
        t = build_distance_tables(book).tables
        arrays[f"b{i}_tables_sha256"] = np.array(hashlib.sha256(t.tobytes()).hexdigest())
        pick = np.random.default_rng(i).integers(0, [m, l_count, l_count], size=(256, 3))
        arrays[f"b{i}_pick"] = pick
        arrays[f"b{i}_values"] = t[pick[:, 0], pick[:, 1], pick[:, 2]]
    rng = np.random.default_rng(8)
    sizes = [1, 2, 7, 8, 9, 100, 128, 129, 255, 256, 1000, 8191, 8193, 20001]
    for n in sizes:
        x = rng.random(n) * 10.0 ** rng.integers(-3, 6, size=n)
        arrays[f"m{n}_x"] = x
        arrays[f"m{n}_mean"] = np.array([np.mean(np.sqrt(x)), np.mean(x)])
    arrays["sizes"] = np.array(sizes)
    save("tables_mean", **arrays)


def make_train():
    """Reference train_codebook (pq.py:155-202), incl. empty-codeword reseeds."""
    arrays = {}
    rng = np.random.default_rng(77)
    x0 = rng.normal(size=(2000, 16)).astype(np.float32)
    arrays.update(t0_x=x0, t0_book=train_codebook(x0, 4, 32, iterations=5, seed=3).codewords,
                  t0_args=np.array([4, 32, 5, 3]))
    # many duplicated rows: codewords go empty and are re-seeded on the farthest points
    rows = rng.normal(size=(40, 12)).astype(np.float32) * 3
    x1 = rows[rng.integers(0, 40, size=300)]
    arrays.update(t1_x=x1, t1_book=train_codebook(x1, 2, 64, iterations=6, seed=5).codewords,
                  t1_args=np.array([2, 64, 6, 5]))
    x2 = (rng.normal(size=(1500, 64)) * 10).astype(np.float32)
    arrays.update(t2_x=x2, t2_book=train_codebook(x2, 1, 256, iterations=3, seed=9).codewords,
                  t2_args=np.array([1, 256, 3, 9]))
    arrays["ncases"] = np.array(3)
    save("train", **arrays)


def make_baselines():
    """Reference cluster_means / original_space_error (baselines.py:26-37, 385-413)."""
    from pqclust.baselines import cluster_means, original_space_error

    arrays = {}
    rng = np.random.default_rng(91)
    cases = [(600, 128, 37, 1.0), (777, 32, 5, 1e3), (800, 40, 300, 1e-3), (130, 7, 3, 10.0), (1, 3, 1, 1.0),
             (300, 200, 9, 1.0)]
    for i, (n, d, k, scale) in enumerate(cases):
        x = (rng.normal(size=(n, d)) * scale + rng.uniform(-5, 5, size=d) * scale).astype(np.float32)
        lab = rng.integers(0, k, size=n)
        if k > 4:
            lab[lab == 2] = 3  # an empty cluster in the middle
        arrays[f"b{i}_x"] = x
        arrays[f"b{i}_labels"] = lab.astype(np.int64)
        arrays[f"b{i}_k"] = np.array(k)
        arrays[f"b{i}_means"] = cluster_means(x.astype(np.float64), lab, k)
        arrays[f"b{i}_means32"] = cluster_means(x, lab, k)
        arrays[f"b{i}_err"] = np.array(original_space_error(x, lab))
    arrays["ncases"] = np.array(len(cases))
    save("baselines", **arrays)


def make_bkmeans():
    """Reference train_binarizer / binarize / hamming_to_centers / majority_center /
    bkmeans_fit (baselines.py:157-382)."""
    from pqclust.baselines import binarize, bkmeans_fit, hamming_to_centers, train_binarizer

    arrays = {}
    rng = np.random.default_rng(93)
    # binarizers and binarized vectors (incl. a zero vector: every bit set)
    for i, (dim, bits, n) in enumerate([(128, 32, 400), (24, 16, 50), (64, 64, 200), (40, 40, 30)]):
        bz = train_binarizer(dim, bits, seed=10 + i)
        x = (rng.normal(size=(n, dim)) * 7).astype(np.float32)
        x[0] = 0.0
        arrays[f"z{i}_rot"] = bz.rotation
        arrays[f"z{i}_args"] = np.array([dim, bits, 10 + i])
        arrays[f"z{i}_x"] = x
        arrays[f"z{i}_codes"] = binarize(bz, x)
    arrays["nbin"] = np.array(4)
    # Hamming matrix
    a = rng.integers(0, 256, size=(40, 5), dtype=np.uint8)
    b = rng.integers(0, 256, size=(9, 5), dtype=np.uint8)
    arrays.update(h_a=a, h_b=b, h_d=hamming_to_centers(a, b))
    # fits: clustered codes (noisy copies of prototypes), duplicates forcing repairs, ties
    fits = []
    protos = rng.integers(0, 256, size=(12, 4), dtype=np.uint8)
    noise = (rng.random(size=(900, 32)) < 0.08).astype(np.uint8)
    codes0 = protos[rng.integers(0, 12, size=900)] ^ np.packbits(noise, axis=1)
    fits.append((codes0, 12, 15, 3, None))
    dup = np.repeat(rng.integers(0, 256, size=(6, 2), dtype=np.uint8), 20, axis=0)
    fits.append((dup, 10, 6, 1, None))  # 6 distinct codes, K=10: empty clusters every iteration
    codes2 = rng.integers(0, 256, size=(500, 8), dtype=np.uint8)
    fits.append((codes2, 30, 8, 5, None))
    ties = np.array([[0x00], [0x0F], [0xF0], [0xFF], [0x3C], [0xC3]] * 5, dtype=np.uint8)
    fits.append((ties, 3, 5, 0, np.array([[0x00], [0xFF], [0x0F]], dtype=np.uint8)))
    codes4 = rng.integers(0, 256, size=(300, 16), dtype=np.uint8)
    fits.append((codes4, 7, 4, 2, None))
    for i, (codes, k, it, seed, init) in enumerate(fits):
        res = bkmeans_fit(codes, k, max_iterations=it, seed=seed, initial_centers=init)
        arrays[f"f{i}_codes"] = codes
        arrays[f"f{i}_args"] = np.array([k, it, seed])
        arrays[f"f{i}_init"] = init if init is not None else np.zeros((0, codes.shape[1]), np.uint8)
        arrays[f"f{i}_centers"] = res.centers
        arrays[f"f{i}_labels"] = res.labels
        arrays[f"f{i}_obj"] = np.array([s.objective for s in res.trace])
        arrays[f"f{i}_obj_sq"] = np.array([s.objective_sq for s in res.trace])
        arrays[f"f{i}_rep"] = np.array([s.repaired_clusters for s in res.trace])
        arrays[f"f{i}_conv"] = np.array(res.converged)
    arrays["nfit"] = np.array(len(fits))
    save("bkmeans", **arrays)


def make_io():
    """Bytes of files written by the reference's io writers (io.py), and their inputs."""
    import tempfile

    from pqclust import io as rio

    rng = np.random.default_rng(95)
    vec = (rng.normal(size=(37, 12)) * 3).astype(np.float32)
    bvec = rng.integers(0, 256, size=(19, 7)).astype(np.float32)
    codes = rng.integers(0, 200, size=(53, 6)).astype(np.uint8)
    book = PQCodebook(rng.normal(size=(3, 16, 4)).astype(np.float32))
    packed = rng.integers(0, 256, size=(23, 3), dtype=np.uint8)
    labels = rng.integers(0, 2**32 - 1, size=41, dtype=np.uint64).astype(np.uint32)
    arrays = dict(vec=vec, bvec=bvec, codes=codes, book=book.codewords, packed=packed, labels=labels)
    with tempfile.TemporaryDirectory() as td:
        writers = {"fvecs": lambda p: rio.write_fvecs(p, vec), "bvecs": lambda p: rio.write_bvecs(p, bvec),
                   "pqkc": lambda p: rio.write_codes(p, codes, 200), "pqcb": lambda p: rio.write_codebook(p, book),
                   "pqkb": lambda p: rio.write_binary_codes(p, packed), "labels": lambda p: rio.write_labels(p, labels)}
        for name, write in writers.items():
            path = Path(td) / name
            write(path)
            arrays[f"file_{name}"] = np.frombuffer(path.read_bytes(), dtype=np.uint8).copy()
    save("io", **arrays)


if __name__ == "__main__":
    makers = {"assign": make_assign, "fit": make_fit, "encode": make_encode, "vote": make_vote,
              "tables_mean": make_tables_and_mean, "config1": make_config1, "train": make_train,
              "baselines": make_baselines, "bkmeans": make_bkmeans, "io": make_io}
    for name in sys.argv[1:] or list(makers):  # default: regenerate every fixture
        makers[name]()

"""Small workload that launches every hot kernel of the path once or twice, checked
against the oracle and (PQK_GUARD=1) for out-of-bounds stores:

  PQK_GUARD=1 python tools/sanitize_fit.py                       # atomic histogram
  PQK_GUARD=1 PQK_HIST_MODE=tiled python tools/sanitize_fit.py   # cluster-tiled hbin_*

With PQK_GUARD=1 every buffer the engine hands to a kernel for writing sits between two
64 KB guard zones of 0xA5 (engine._alloc), and the run fails if any zone changed.  (The
pool does not allow compute-sanitizer; this is the substitute, plus the oracle checks.)

Covered: dedup, scale preparation, the 8-bit (hscan8/hfinal8) and 16-bit (hscan/hfinal)
first tiers, the fp32 scan and its list tier, the exact rescans, histogram (atomic and
cluster-tiled hbin_*), counts, vote (tcgen05 vote_tc + fp64/double-double stages),
objective tree, repair (radix select + bitonic sort), the tcgen05 encoders (encode_tc,
encode_tck) with the fp64 fallback, codebook training and the table builder.  Results are
checked against the oracle, so a silent corruption also fails the run."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1709_03708_b200 as pqk  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402
from paper_1709_03708_b200 import _lib  # noqa: E402

sys.path.insert(0, "tests")
from helpers import lattice_tables, mixture_codes, random_tables  # noqa: E402

lib = _lib.load()
rng = np.random.default_rng(4)
fails = 0


def check(name, ok):
    global fails
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    fails += 0 if ok else 1


# assignment tiers: mode 2 (8-bit at M=4 / 16-bit at M=8), 3 (+ fp32 list tier), 4 (16-bit at M=4), 1 (fp32)
for m, mode in ((4, 2), (4, 3), (4, 4), (4, 5), (8, 2), (8, 3), (4, 1)):
    tables = random_tables(m, 256, seed=m, sub_dim=4)
    codes = mixture_codes(6000, m, 256, 80, seed=m + mode)
    centers = codes[rng.choice(len(codes), size=300, replace=False)].copy()
    centers[rng.integers(0, 300, size=40)] = centers[5]  # duplicates
    _lib.check(lib.pqk_set_scan_mode(mode), "scan mode")
    try:
        labels = pqk.assign(codes, centers, tables)
    finally:
        _lib.check(lib.pqk_set_scan_mode(0), "scan mode")
    check(f"assign m={m} mode={mode}", np.array_equal(labels, O.assign_c(codes, centers, tables)))

# ties across chunks (lattice tables), 8-bit tier
tables = lattice_tables(4, 8)
codes = rng.integers(0, 8, size=(3000, 4)).astype(np.uint8)
centers = rng.integers(0, 8, size=(200, 4)).astype(np.uint8)
_lib.check(lib.pqk_set_scan_mode(2), "scan mode")
try:
    labels = pqk.assign(codes, centers, tables)
finally:
    _lib.check(lib.pqk_set_scan_mode(0), "scan mode")
check("assign lattice 8-bit", np.array_equal(labels, O.assign_c(codes, centers, tables)))

# fits with repairs (K close to the number of distinct codes); the histogram path is the
# one PQK_HIST_MODE selects for the process (run once with PQK_HIST_MODE=tiled for hbin_*)
tables = random_tables(4, 256, seed=9, sub_dim=4)
codes = mixture_codes(8000, 4, 256, 50, seed=9)
_lib.check(lib.pqk_set_scan_mode(2), "scan mode")
try:
    res = pqk.fit(codes, tables, 400, max_iterations=4, seed=2)
finally:
    _lib.check(lib.pqk_set_scan_mode(0), "scan mode")
ref = O.fit(codes, tables, 400, max_iterations=4, seed=2, scan=O.assign_c)
check("fit m=4 (repairs)", np.array_equal(res.labels, ref["labels"]) and np.array_equal(res.centers, ref["centers"]))
tables16 = random_tables(16, 256, seed=16, sub_dim=2)
codes16 = mixture_codes(4000, 16, 256, 60, seed=16)
res = pqk.fit(codes16, tables16, 100, max_iterations=3, seed=5)
ref = O.fit(codes16, tables16, 100, max_iterations=3, seed=5, scan=O.assign_c)
check("fit m=16", np.array_equal(res.labels, ref["labels"]) and np.array_equal(res.centers, ref["centers"]))

# encoders: dsub 32 (encode_tc), dsub 512 (encode_tck), fp64 fallback via ties
book = rng.normal(size=(4, 256, 32)).astype(np.float32)
x = rng.normal(size=(3000, 128)).astype(np.float32)
x[:50] = np.concatenate([book[m][7] for m in range(4)])[None, :]  # exact codewords
check("encode dsub=32", np.array_equal(pqk.encode(pqk.PQCodebook(book), x), O.encode(book, x)))
book3 = rng.normal(size=(2, 256, 512)).astype(np.float32)
x3 = rng.normal(size=(600, 1024)).astype(np.float32)
check("encode dsub=512", np.array_equal(pqk.encode(pqk.PQCodebook(book3), x3), O.encode(book3, x3)))

# codebook training + tables
sample = rng.normal(size=(3000, 16)).astype(np.float32)
cb = pqk.train_codebook(sample, 2, 256, iterations=3, seed=1)
ref_cb = O.train_codebook(sample, 2, 256, iterations=3, seed=1)
check("train_codebook", np.array_equal(np.asarray(cb.codewords), np.asarray(ref_cb)))
t_gpu = pqk.build_distance_tables(cb).tables
check("build_distance_tables", np.array_equal(t_gpu, O.build_distance_tables(np.asarray(cb.codewords))))

# a mid-size assignment: several persistent passes per CTA, 8-bit tier by default size rule
tables = random_tables(4, 256, seed=21, sub_dim=4)
codes = mixture_codes(400_000, 4, 256, 3000, seed=21)
centers = codes[rng.choice(len(codes), size=6000, replace=False)].copy()
labels = pqk.assign(codes, centers, tables)
check("assign 4e5 x 6e3 default tiers", np.array_equal(labels, O.assign_c(codes, centers, tables)))

from paper_1709_03708_b200 import engine  # noqa: E402

if engine._GUARD:
    bad = engine.check_guards()
    check(f"guard zones intact ({len(engine._GUARDS)} guarded buffers)", not bad)
print("SANITIZE_FIT", "OK" if not fails else f"{fails} MISMATCHES", flush=True)
sys.exit(1 if fails else 0)

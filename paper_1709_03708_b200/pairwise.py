"""numpy pairwise-summation tree: shard split and combine (host logic).

``np.mean`` (clustering.py:448-449) sums float64 with numpy's pairwise tree
(numpy/_core/src/umath/loops_utils.h.src): n <= 128 is a leaf, otherwise
n2 = n//2 - (n//2 % 8) and sum(a[:n2]) + sum(a[n2:]).  The subtree over a slice
depends only on its length, so a device (or a rank) can sum the subtree of its
slice with the plan for that length.  Sharding codes along the tree's top-level
splits lets every rank sum its subtree locally; :func:`combine` then adds the
partials in the tree's order, reproducing numpy's float64 result exactly.
"""

from __future__ import annotations


def _split(n: int) -> int:
    n2 = n // 2
    return n2 - (n2 % 8)


def tree_split(n: int, parts: int) -> list[tuple[int, int]]:
    """(offset, length) of `parts` contiguous shards aligned to tree nodes.

    Parts are split recursively: a node with p parts gives ceil(p/2) to its left
    child and floor(p/2) to its right child; a leaf that still has p > 1 parts
    goes whole to the first part and the rest are empty.
    """
    out: list[tuple[int, int]] = []

    def rec(off: int, length: int, p: int) -> None:
        if p == 1:
            out.append((off, length))
            return
        if length <= 128:
            out.append((off, length))
            out.extend((off + length, 0) for _ in range(p - 1))
            return
        n2 = _split(length)
        pl = (p + 1) // 2
        rec(off, n2, pl)
        rec(off + n2, length - n2, p - pl)

    rec(0, n, parts)
    return out


def tree_combine(n: int, partials: list[float]) -> float:
    """Combine per-shard subtree sums (from tree_split(n, len(partials))) in tree order."""
    it = iter(range(len(partials)))

    def rec(length: int, p: int) -> float:
        if p == 1:
            return float(partials[next(it)])
        if length <= 128:
            v = float(partials[next(it)])
            for _ in range(p - 1):
                next(it)
            return v
        n2 = _split(length)
        pl = (p + 1) // 2
        left = rec(n2, pl)
        right = rec(length - n2, p - pl)
        return left + right

    return rec(n, len(partials))

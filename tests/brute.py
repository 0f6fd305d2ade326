"""Brute-force restatements of the paper's definitions, for tiny inputs only (pins for the oracle).

Written independently of oracle.c and in a different style: strings instead of codes, the
"multiply the repeated diet pattern with the sequence" formulation of P:282, segments obtained by
splitting at N, canonical k-mers compared as strings, windows enumerated as Python sets, and the
hash written in its multiplicative form with Python big integers.
"""
from __future__ import annotations

COMP = {"A": "T", "C": "G", "G": "C", "T": "A"}
VAL = {"A": 0, "C": 1, "G": 2, "T": 3}


def diet(pattern: str, L: int, s: int):
    """The repeated pattern shifted right by s (P:286 (1)): 0 before the shift."""
    p = len(pattern)
    return [1 if (i >= s and pattern[(i - s) % p] == "1") else 0 for i in range(L)]


def sparsify_str(seq: str, pattern: str, s: int):
    d = diet(pattern, len(seq), s)
    kept = [(i, seq[i]) for i in range(len(seq)) if d[i]]
    return "".join(b for _, b in kept), [i for i, _ in kept]


def norm(b: str) -> str:
    b = b.upper()
    return b if b in "ACGT" else "N"


def wang_hash_bigint(x: int, k: int) -> int:
    """Thomas Wang's 64-bit mix (ref. 120) with each step mod 4^k, multiplicative form."""
    m = 4 ** k
    x = (x * (2 ** 21 - 1) - 1) % m
    x = x ^ (x >> 24)
    x = (x * 265) % m
    x = x ^ (x >> 14)
    x = (x * 21) % m
    x = x ^ (x >> 28)
    x = (x * (2 ** 31 + 1)) % m
    return x


def kmer_value(s: str) -> int:
    v = 0
    for c in s:
        v = v * 4 + VAL[c]
    return v


def revcomp(s: str) -> str:
    return "".join(COMP[c] for c in reversed(s))


def brute_minimizers(seq: str, pattern: str, s: int, k: int, w: int, pos_base: int = 0):
    """Set-union over windows of the all-ties window minima; returns sorted [(hash, pos, strand)]."""
    seq = "".join(norm(b) for b in seq)
    sub, orig = sparsify_str(seq, pattern, s)
    # split the patterned sequence at N into N-free segments, remembering original positions
    segs, cur = [], []
    for c, o in zip(sub, orig):
        if c == "N":
            segs.append(cur)
            cur = []
        else:
            cur.append((c, o))
    segs.append(cur)
    out = set()
    for seg in segs:
        letters = "".join(c for c, _ in seg)
        items = []
        for j in range(len(seg) - k + 1):
            f = letters[j:j + k]
            r = revcomp(f)
            if f == r:
                items.append(None)                      # palindrome: never a window minimum
            else:
                canon = min(f, r)                       # A<C<G<T string order == numeric order
                items.append((wang_hash_bigint(kmer_value(canon), k), pos_base + seg[j][1], int(f > r)))
        n = len(items)
        if n == 0:
            continue
        wins = [items[a:a + w] for a in range(n - w + 1)] if n >= w else [items]
        for W in wins:
            vals = [it[0] for it in W if it is not None]
            if not vals:
                continue
            mn = min(vals)
            out |= {it for it in W if it is not None and it[0] == mn}
    return sorted(out, key=lambda t: t[1])


def true_phases(pattern: str, g: int, L: int, strand: int):
    """All shifts s that put an error-free read of reference [g, g+L) (or its reverse complement)
    in register with the reference's phase-0 patterned genome: included read index i <-> included
    reference position, for every i >= s.  Brute force over s (used for GIVEN-mode invariants)."""
    p = len(pattern)
    ok = []
    for s in range(p):
        good = True
        for i in range(s, min(L, s + 4 * p)):
            u = g + i if not strand else g + L - 1 - i
            if (pattern[(i - s) % p] == "1") != (pattern[u % p] == "1"):
                good = False
                break
        if good:
            ok.append(s)
    return ok

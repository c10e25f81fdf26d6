#!/usr/bin/env python3
"""Shared-memory bank model of the element kernels' line contractions, and the
search that produced `kFaceRot6` (paper_2008_04356_b200/csrc/kernels.cu).

Model (B200, 64-bit shared loads): a warp's load is served half-warp by
half-warp; within a half-warp the 16 threads' 8-byte words fall on 16 banks
(word index mod 16); threads reading the same word are served together
(broadcast); the cost of a half-warp is the largest number of distinct words on
one bank.  ncu's "ideal" for such a load is 2 wavefronts per warp.

  tools/bank_rotation.py            print the cost tables (unrotated / shipped)
  tools/bank_rotation.py --search   redo the N+1 = 6 per-half-warp search

The element block is [row][node], node = (i * N1 + j) * N1 + k.  A face thread
it = side * N2 + a * N1 + b reads the N1 nodes of its line (along i, j or k for
sides 0-1, 2-3, 4-5) in the order m -> (m + rot) mod N1.
"""
from __future__ import annotations

import os
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KERNELS = os.path.join(HERE, "..", "paper_2008_04356_b200", "csrc", "kernels.cu")


def half_warp_cost(words):
    """Wavefronts of one half-warp: max distinct words per bank."""
    banks = {}
    for w in set(words):
        banks.setdefault(w % 16, set()).add(w)
    return max(len(v) for v in banks.values()) if banks else 0


def face_line(n1, it):
    """(base, stride) of the line a face thread reads."""
    n2 = n1 * n1
    side, f = divmod(it, n2)
    a, b = divmod(f, n1)
    d = side >> 1
    if d == 0:
        return a * n1 + b, n2
    if d == 1:
        return a * n2 + b, n1
    return (a * n1 + b) * n1, 1


def shipped_face_rot6():
    src = open(KERNELS).read()
    body = re.search(r"kFaceRot6\[216\] = \{(.*?)\};", src, re.S).group(1)
    body = re.sub(r"//[^\n]*", "", body)
    tab = [int(x) for x in re.findall(r"\d+", body)]
    assert len(tab) == 216
    return tab


def face_rot(n1, it, table6=None):
    """The rotation face_rot<N1> of kernels.cu."""
    n2 = n1 * n1
    side, f = divmod(it, n2)
    a, b = divmod(f, n1)
    d = side >> 1
    if n1 == 4:
        return 0 if d == 0 else a
    if n1 == 8:
        return 0 if d == 0 else ((a & 1) if d == 1 else (b >> 1) + 4 * (a & 1))
    if n1 == 6:
        return table6[it]
    return 0


def prolong_cost(n1, rot, index=lambda n: n):
    """Wavefronts of prolonging one row on all 6 * N2 face nodes; ideal = N1 * half-warps."""
    n2 = n1 * n1
    total = 0
    for h0 in range(0, 6 * n2, 16):
        its = range(h0, min(h0 + 16, 6 * n2))
        for m in range(n1):
            words = []
            for it in its:
                base, stride = face_line(n1, it)
                words.append(index(base + ((m + rot(it)) % n1) * stride))
            total += half_warp_cost(words)
    return total, n1 * ((6 * n2 + 15) // 16)


def node_rot(n1, t):
    """node_rot<N1> of kernels.cu."""
    return 1 if n1 == 6 and (t & ~15) < 36 * (t // 36) else 0


def volume_cost(n1, d, rot):
    """Wavefronts of one row of the node threads' contraction along direction d."""
    n2, n3 = n1 * n1, n1 ** 3
    total = 0
    for h0 in range(0, n3, 16):
        for m in range(n1):
            words = []
            for t in range(h0, min(h0 + 16, n3)):
                i, j, k = t // n2, (t // n1) % n1, t % n1
                mr = (m + rot(t)) % n1
                words.append((j * n1 + k + mr * n2) if d == 0 else ((i * n2 + k + mr * n1) if d == 1 else (i * n1 + j) * n1 + mr))
            total += half_warp_cost(words)
    return total, n1 * ((n3 + 15) // 16)


def swz(n1, n):
    """swz<N1> of kernels.cu (k_gradient_ws blocks)."""
    if n1 == 8:
        i, j = n >> 6, (n >> 3) & 7
        return n ^ ((i & 1) << 3) ^ j
    if n1 == 4:
        i = n >> 4
        return n ^ (i << 2) ^ i
    return n


def line_task_cost(n1, d, index=lambda n: n):
    """Wavefronts of one pass of the line tasks of direction d (16 consecutive lines per half-warp)."""
    n2 = n1 * n1
    total = 0
    for f0 in range(0, n2, 16):
        for m in range(n1):
            words = []
            for f in range(f0, min(f0 + 16, n2)):
                base, stride = face_line(n1, 2 * d * n2 + f)
                words.append(index(base + m * stride))
            total += half_warp_cost(words)
    return total, n1 * ((n2 + 15) // 16)


def search_half_warp(n1, its, budget, limit=400000):
    """Depth-first assignment of rotations to the threads of one half-warp with total cost <= budget."""
    banks = [dict() for _ in range(n1)]
    rots = [0] * len(its)
    visited = [0]

    def cost():
        return sum(max((len(v) for v in banks[m].values()), default=0) for m in range(n1))

    def rec(i):
        visited[0] += 1
        if visited[0] > limit:
            return False
        if i == len(its):
            return True
        base, stride = face_line(n1, its[i])
        for r in range(n1):
            added = []
            for m in range(n1):
                w = base + ((m + r) % n1) * stride
                s = banks[m].setdefault(w % 16, set())
                if w not in s:
                    s.add(w)
                    added.append((m, w))
            if cost() <= budget and rec(i + 1):
                rots[i] = r
                return True
            for m, w in added:
                banks[m][w % 16].discard(w)
        return False

    return rots if rec(0) else None


def search6():
    table = []
    for h0 in range(0, 216, 16):
        its = list(range(h0, min(h0 + 16, 216)))
        for budget in range(6, 24):
            r = search_half_warp(6, its, budget)
            if r is not None:
                break
        table += r
    return table


def main():
    if "--search" in sys.argv:
        tab = search6()
        print("cost", prolong_cost(6, lambda it: tab[it]))
        for s in range(6):
            print("    " + ", ".join(str(x) for x in tab[s * 36:(s + 1) * 36]) + ",  // side %d" % s)
        return
    tab6 = shipped_face_rot6()
    for n1 in (4, 6, 8):
        plain, ideal = prolong_cost(n1, lambda it: 0)
        rotated, _ = prolong_cost(n1, lambda it: face_rot(n1, it, tab6))
        print(f"N+1 = {n1}: face prolongation of one row: unrotated {plain}, rotated {rotated}, ideal {ideal} wavefronts")
        for d in range(3):
            v0, vi = volume_cost(n1, d, lambda t: 0)
            v1, _ = volume_cost(n1, d, lambda t: node_rot(n1, t))
            l0, li = line_task_cost(n1, d)
            l1, _ = line_task_cost(n1, d, lambda n: swz(n1, n))
            print(f"   direction {d}: node-thread contraction {v0} -> {v1} (ideal {vi}); line tasks {l0} -> swizzled {l1} (ideal {li})")


if __name__ == "__main__":
    main()

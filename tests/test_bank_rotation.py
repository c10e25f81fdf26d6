"""Shared-memory bank model of the line contractions (tools/bank_rotation.py):
the shipped rotation table, closed forms and swizzles of csrc/kernels.cu do what
DESIGN.md §4d says they do.  CPU only; the kernels' results are covered by the
GPU parity tests, which run the rotated order."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tools"))
import bank_rotation as B  # noqa: E402


def test_face_rotation_table_is_a_rotation_and_cuts_the_conflicts():
    tab = B.shipped_face_rot6()
    assert len(tab) == 216 and all(0 <= r < 6 for r in tab)
    plain, ideal = B.prolong_cost(6, lambda it: 0)
    rotated, _ = B.prolong_cost(6, lambda it: tab[it])
    assert (plain, ideal) == (152, 84)
    assert rotated <= 96


def test_closed_form_rotations_are_conflict_free():
    for n1 in (4, 8):
        plain, ideal = B.prolong_cost(n1, lambda it: 0)
        rotated, _ = B.prolong_cost(n1, lambda it: B.face_rot(n1, it))
        assert plain > 2 * ideal
        assert rotated == ideal


def test_node_thread_rotation():
    for d, want in ((0, 88), (1, 84), (2, 84)):
        plain, ideal = B.volume_cost(6, d, lambda t: 0)
        rotated, _ = B.volume_cost(6, d, lambda t: B.node_rot(6, t))
        assert ideal == 84 and rotated <= want <= plain
    for n1 in (4, 8):  # whole half-warps per plane: nothing to rotate
        for d in range(3):
            plain, ideal = B.volume_cost(n1, d, lambda t: 0)
            assert plain == ideal


def test_swizzle_is_a_bijection_and_conflict_free():
    for n1 in (4, 8):
        n3 = n1 ** 3
        assert sorted(B.swz(n1, n) for n in range(n3)) == list(range(n3))
        for d in range(3):
            cost, ideal = B.line_task_cost(n1, d, lambda n: B.swz(n1, n))
            assert cost == ideal
        cost, ideal = B.prolong_cost(n1, lambda it: 0, lambda n: B.swz(n1, n))
        assert cost == ideal
        # node rows (thread t reads node t)
        for h0 in range(0, n3, 16):
            assert B.half_warp_cost([B.swz(n1, t) for t in range(h0, h0 + 16)]) == 1

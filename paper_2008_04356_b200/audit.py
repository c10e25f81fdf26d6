"""Communication audit of a multi-rank run.

Checks the three claims of the reference's audit (audit_communication,
/root/reference/proj/src/audit.cpp:44-148) on the traces the B200 path
records (sdg_trace_json):
  1. the rank-map exchange is the only collective and stays in the init phase;
  2. every simulation-phase message is pure face / mortar data whose size is a
     whole number of face-node blocks and matches the partition's halo plan;
  3. sliding-mesh messages only connect ranks on opposite sides of an
     interface, and every send is matched by the partner's receive.
"""
from __future__ import annotations

from collections import defaultdict

from . import capi
from . import types as T

INIT, SOL_CONF, SOL_MORTAR, LIFT_MORTAR, FVN_CONF, GRAD_MORTAR, FLUX_MORTAR = 1, 2, 3, 5, 6, 7, 9
NCOMP = {SOL_CONF: 5, SOL_MORTAR: 5, LIFT_MORTAR: 4, FVN_CONF: 4, GRAD_MORTAR: 12, FLUX_MORTAR: 5}
CONF = {SOL_CONF, FVN_CONF}
MORTAR = {SOL_MORTAR, LIFT_MORTAR, GRAD_MORTAR, FLUX_MORTAR}


def _band_of(mesh: T.MeshSpec, gid: int) -> int:
    off = 0
    for b in range(mesh.n_bands):
        n = mesh.bands[b].nx * mesh.ny * mesh.nz
        if gid < off + n:
            return b
        off += n
    raise ValueError(gid)


def audit(traces: list[dict], mesh: T.MeshSpec) -> dict:
    n_ranks = traces[0]["n_ranks"]
    n2 = traces[0]["n1"] ** 2
    rep = dict(passed=True, violations=[], init_collective_sends=0, post_init_collectives=0, data_messages=0,
               data_bytes=0)

    def fail(msg):
        rep["passed"] = False
        rep["violations"].append(msg)

    plans = [capi.plan(mesh, n_ranks, r) for r in range(n_ranks)]
    halo = {(p["rank"], h["partner"]): len(h["keys"]) for p in plans for h in p["halo"]}
    bands_of = [{_band_of(mesh, g) for g in p["elements"]} for p in plans]
    vg = [mesh.bands[b].vg_y for b in range(mesh.n_bands)]
    sliding_pairs = set()
    nb = mesh.n_bands
    for b in range(nb if mesh.periodic_x else nb - 1):
        l, r = b, (b + 1) % nb
        if nb > 1 and vg[l] != vg[r]:
            sliding_pairs.add((l, r))
            sliding_pairs.add((r, l))
    sends, recvs = defaultdict(list), defaultdict(list)
    for tr in traces:
        for step, stage, src, dst, nbytes, kind, is_send in tr["rows"]:
            if kind == INIT:
                if step < 0:
                    rep["init_collective_sends"] += is_send
                else:
                    rep["post_init_collectives"] += 1
                    fail(f"collective outside the init phase at step {step} stage {stage} ({src}->{dst})")
                continue
            if kind not in NCOMP:
                fail(f"unknown message kind {kind}")
                continue
            block = 8 * n2 * NCOMP[kind]
            if nbytes <= 0 or nbytes % block:
                fail(f"kind {kind} message of {nbytes} B is not a whole number of face-node blocks")
            if kind in CONF and nbytes != halo.get((src, dst), -1) * block:
                fail(f"conforming message {src}->{dst} of {nbytes} B does not match the halo plan")
            if kind in MORTAR and not any((a, b) in sliding_pairs for a in bands_of[src] for b in bands_of[dst]):
                fail(f"mortar message between ranks {src} and {dst} that share no sliding interface")
            key = (step, stage, kind, src, dst)
            (sends if is_send else recvs)[key].append(nbytes)
            if is_send:
                rep["data_messages"] += 1
                rep["data_bytes"] += nbytes
    if sends != recvs:
        fail("sends and receives do not pair up")
    return rep

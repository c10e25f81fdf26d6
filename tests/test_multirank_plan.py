"""N>1 host logic on CPU with gloo, world_size 2..8 (no GPU): every rank builds
its own partition / halo / mortar message plan (what the NCCL rounds of
solver.cu exchange), the plans are all-gathered over gloo, and every pair of
ranks must derive matching blocks independently — the stamp check of
proj/tests/test_partition.cpp:184-227 extended to the conforming halo.
Partition rules follow proj/src/partition.cpp:17-83 (no rank on both sides of
a sliding interface)."""
import math
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2008_04356_b200 import capi
from paper_2008_04356_b200 import types as T


def meshes():
    L = 2 * math.pi
    return {
        "tgv3": T.mesh_spec([(3, 1.0, 0.0), (4, 1.0, 0.2), (3, 1.0, 0.0)], ny=4, nz=3, width=L, height=L, depth=L),
        "box0": T.mesh_spec([(4, 1.0, 0.0), (4, 1.0, 0.5)], ny=4, nz=4, periodic=(False, True, True)),
        "bands5": T.mesh_spec([(2, 1.0, 0.0), (3, 1.0, 1.0), (2, 2.0, 0.0), (2, 1.0, 0.0), (2, 1.0, 0.7)], ny=5, nz=2),
        "tgv3_sfc": T.mesh_spec([(3, 1.0, 0.0), (4, 1.0, 0.2), (3, 1.0, 0.0)], ny=4, nz=3, width=L, height=L, depth=L,
                                partition=T.PARTITION_SFC),
        "box0_sfc": T.mesh_spec([(4, 1.0, 0.0), (4, 1.0, 0.5)], ny=4, nz=4, periodic=(False, True, True),
                                partition=T.PARTITION_SFC),
        "tgv3_yslab": T.mesh_spec([(3, 1.0, 0.0), (4, 1.0, 0.2), (3, 1.0, 0.0)], ny=8, nz=3, width=L, height=L,
                                  depth=L, partition=T.PARTITION_YSLAB),
    }


def check_plans(plans, n_ranks, mesh):
    by_rank = {p["rank"]: p for p in plans}
    elems = [g for p in plans for g in p["elements"]]
    assert len(elems) == len(set(elems))
    total = sum(mesh.bands[b].nx for b in range(mesh.n_bands)) * mesh.ny * mesh.nz
    assert sorted(elems) == list(range(total))
    for a in range(n_ranks):
        for h in by_rank[a]["halo"]:
            b = h["partner"]
            assert b != a
            back = [x for x in by_rank[b]["halo"] if x["partner"] == a]
            assert len(back) == 1 and back[0]["keys"] == h["keys"], (a, b)
        for m in by_rank[a]["mortars"]:
            b = m["partner"]
            back = [x for x in by_rank[b]["mortars"] if x["partner"] == a and x["role"] == 1 - m["role"]]
            if a == b:
                back = [x for x in by_rank[a]["mortars"] if x["partner"] == a and x["role"] == 1 - m["role"]]
            assert len(back) == 1 and back[0]["keys"] == m["keys"], (a, b, m["role"])
    if n_ranks > 1 and mesh.partition != T.PARTITION_YSLAB:
        for p in plans:
            roles = {m["role"] for m in p["mortars"]}
            selfs = [m for m in p["mortars"] if m["partner"] == p["rank"]]
            assert not selfs, "a rank may not own both sides of a sliding interface"
            assert len(roles) <= 2


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = []
    for name, mesh in meshes().items():
        for delta in (0.0, 0.37, 1.0, 2.9):
            try:
                mine = capi.plan(mesh, world, rank, delta)
            except T.ConfigError:  # e.g. 3 ranks over 5 bands (partition.cpp:31-46): same on every rank
                continue
            allp = [None] * world
            dist.all_gather_object(allp, mine)
            check_plans(allp, world, mesh)
            ok.append((name, delta))
    dist.barrier()
    dist.destroy_process_group()
    results[rank] = len(ok)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_plans_agree_across_gloo_ranks(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    res = mgr.dict()
    procs = [ctx.Process(target=_worker, args=(r, world, PORTS[world], res))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert len(res) == world and len(set(res.values())) == 1


PORTS = {2: free_port(), 3: free_port()}


@pytest.mark.parametrize("world", [1, 2, 4, 6, 8])
def test_plans_agree_in_process(world):
    for mesh in meshes().values():
        for delta in (0.0, 0.37, 1.0):
            try:
                plans = [capi.plan(mesh, world, r, delta) for r in range(world)]
            except T.ConfigError:
                continue
            check_plans(plans, world, mesh)


def test_two_ranks_over_three_bands_split_static_moving():
    mesh = meshes()["tgv3"]
    p0, p1 = capi.plan(mesh, 2, 0), capi.plan(mesh, 2, 1)
    assert len(p0["elements"]) == 2 * 3 * 4 * 3 and len(p1["elements"]) == 4 * 4 * 3


def test_sfc_partition_reduces_the_halo():
    """Space-filling-curve split inside a band: same elements per rank, fewer
    halo faces than lexicographic slabs when a band is cut into many parts."""
    def halo_faces(partition):
        mesh = T.mesh_spec([(8, 1.0, 0.0), (8, 1.0, 0.5)], ny=8, nz=8, partition=partition)
        plans = [capi.plan(mesh, 8, r) for r in range(8)]
        return sum(len(h["keys"]) for p in plans for h in p["halo"]), [len(p["elements"]) for p in plans]
    lex, n_lex = halo_faces(T.PARTITION_LEX)
    sfc, n_sfc = halo_faces(T.PARTITION_SFC)
    assert n_lex == n_sfc
    assert sfc <= lex


def _neighbours(mesh, g):
    """(band, ix, iy, iz) neighbours of global element g across its 6 sides, with the band
    index of each (a band change means a sliding interface)."""
    nb = [mesh.bands[b].nx for b in range(mesh.n_bands)]
    off = [sum(nb[:b]) * mesh.ny * mesh.nz for b in range(mesh.n_bands)]
    b = max(i for i in range(mesh.n_bands) if off[i] <= g)
    r = g - off[b]
    ix, iy, iz = r // (mesh.ny * mesh.nz), (r // mesh.nz) % mesh.ny, r % mesh.nz
    out = []
    for dx in (-1, 1):
        jb, jx = b, ix + dx
        if jx < 0:
            jb = (b - 1) % mesh.n_bands
            jx = nb[jb] - 1
        elif jx >= nb[b]:
            jb = (b + 1) % mesh.n_bands
            jx = 0
        out.append((jb, off[jb] + (jx * mesh.ny + iy) * mesh.nz + iz))
    for dy in (-1, 1):
        out.append((b, off[b] + (ix * mesh.ny + (iy + dy) % mesh.ny) * mesh.nz + iz))
    for dz in (-1, 1):
        out.append((b, off[b] + (ix * mesh.ny + iy) * mesh.nz + (iz + dz) % mesh.nz))
    return b, out


@pytest.mark.parametrize("partition", [T.PARTITION_LEX, T.PARTITION_SFC, T.PARTITION_YSLAB])
@pytest.mark.parametrize("bands,ranks", [([(8, 1.0, 0.0)], 2), ([(6, 1.0, 0.0), (6, 1.0, 0.3), (6, 1.0, 0.0)], 3),
                                         ([(6, 1.0, 0.0), (6, 1.0, 0.3), (6, 1.0, 0.0)], 6),
                                         ([(5, 1.0, 0.0), (7, 1.0, 0.3)], 4)])
def test_interior_run_has_only_local_conforming_neighbours(bands, ranks, partition):
    """SURVEY §8(e) overlap: the element run whose kernels are launched while the halo
    exchange is in flight must not touch a remote conforming face (mortar data are
    complete before the element kernels); the local order puts every such element
    first, so the run is [0, number of local-only elements)."""
    if partition == T.PARTITION_YSLAB and ranks > 4:
        pytest.skip("y slabs need n_ranks <= ny")
    mesh = T.mesh_spec(bands, ny=4, nz=2, partition=partition)
    plans = [capi.plan(mesh, ranks, r) for r in range(ranks)]
    owner = {g: r for r, p in enumerate(plans) for g in p["elements"]}
    vg = [mesh.bands[b].vg_y for b in range(mesh.n_bands)]
    for r, p in enumerate(plans):
        els = p["elements"]
        local_only = []
        for g in els:
            b, nbs = _neighbours(mesh, g)
            # sliding neighbours (another band moving at another speed) come through mortars
            local_only.append(all(owner[jg] == r for jb, jg in nbs if jb == b or vg[jb] == vg[b]))
        lo, hi = p["interior_run"]
        assert lo == 0 and hi == sum(local_only)
        assert all(local_only[lo:hi]) and not any(local_only[hi:])


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_yslab_partition_balances_every_band(world):
    """Slabs along the sliding direction: every rank owns ny / world rows of every band (equal work for
    any band layout), both sides of the sliding interfaces, and mortars still pair up across ranks."""
    L = 2 * math.pi
    mesh = T.mesh_spec([(3, 1.0, 0.0), (4, 1.0, 0.2), (3, 1.0, 0.0)], ny=8, nz=3, width=L, height=L, depth=L,
                       partition=T.PARTITION_YSLAB)
    plans = [capi.plan(mesh, world, r, 0.37) for r in range(world)]
    check_plans(plans, world, mesh)
    sizes = [len(p["elements"]) for p in plans]
    assert max(sizes) - min(sizes) <= 10 * 3  # one y row of all bands
    if 8 % world == 0:
        assert len(set(sizes)) == 1
    assert any(m["partner"] == p["rank"] for p in plans for m in p["mortars"])  # rank-local mortars

"""CPU tests of the multi-GPU decomposition (host logic + the exchange
protocol over gloo, world_size 2 and 3).  The per-rank local assembly is
stood in for by the CPU oracle here; on GPUs the same exchange runs over
NCCL between libtal_b200 halo pack/accumulate kernels (SlabDomain.step)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_08777_b200.distributed import SlabPartition, exchange_interfaces, slab_bounds
import paper_2403_08777_b200 as tb


def test_slab_bounds_cover():
    for n, w in [(8, 2), (7, 3), (128, 8), (5, 5)]:
        b = slab_bounds(n, w)
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
        assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_local_meshes_are_slices_of_the_global_box(world):
    cells = (3, 2, 7)
    g = tb.generate_box_mesh(*cells)
    elems = 0
    for r in range(world):
        p = SlabPartition(cells, r, world)
        m = p.local_mesh()
        lo, hi = p.node_range
        e0, e1 = p.elem_range
        np.testing.assert_array_equal(m.coords, g.coords[lo:hi])
        np.testing.assert_array_equal(m.connectivity + lo, g.connectivity[e0:e1])
        elems += m.n_elems
        for nbr, ids in p.interfaces().items():
            q = SlabPartition(cells, nbr, world)
            other = q.interfaces()[r]
            np.testing.assert_array_equal(ids + lo, other + q.node_range[0])
    assert elems == g.n_elems


@pytest.mark.parametrize("spec", ["random:1", "taylor-green", "shear:1.5"])
def test_slab_velocity_is_the_global_field(spec):
    cells = (4, 3, 6)
    g = tb.generate_box_mesh(*cells)
    ug = tb.make_velocity(g, spec)
    for r in range(3):
        p = SlabPartition(cells, r, 3)
        lo, hi = p.node_range
        np.testing.assert_array_equal(p.velocity(spec), ug[lo:hi])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cells, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    p = SlabPartition(cells, rank, world)
    m = p.local_mesh()
    u = p.velocity("random:1", m)
    rhs = O.assemble_rsp(m.coords, m.connectivity, u)  # stand-in for the GPU local assembly
    send, recv = {}, {}
    for nbr, ids in p.interfaces().items():
        send[nbr] = torch.from_numpy(rhs[ids].copy())
        recv[nbr] = torch.empty_like(send[nbr])
    exchange_interfaces(p, send, recv)
    for nbr, ids in p.interfaces().items():
        rhs[ids] += recv[nbr].numpy()
    np.save(os.path.join(out_dir, f"rhs_{rank}.npy"), rhs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_interface_exchange_gloo_matches_single_domain(tmp_path, world, oracle):
    cells = (5, 4, 7)
    mp.start_processes(_worker, args=(world, _free_port(), cells, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    g = oracle.box_mesh(*cells)
    ug = oracle.velocity(g.coords, "random:1")
    ref = oracle.assemble_rsp(g.coords, g.connectivity, ug)
    full = np.full_like(ref, np.nan)
    for r in range(world):
        p = SlabPartition(cells, r, world)
        lo, hi = p.node_range
        loc = np.load(tmp_path / f"rhs_{r}.npy")
        mask = p.owned_mask()
        full[lo:hi][mask] = loc[mask]
        # shared planes agree on both sides after the exchange
        for nbr, ids in p.interfaces().items():
            q = SlabPartition(cells, nbr, world)
            other = np.load(tmp_path / f"rhs_{nbr}.npy")[q.interfaces()[r]]
            assert np.abs(loc[ids] - other).max() <= 1e-15 * np.abs(ref).max()
    assert not np.isnan(full).any()
    chk = oracle.compare(full, ref, g.coords, g.connectivity, ug)
    assert chk.passed, chk


# ---------------------------------------------------------------------------
# general meshes: recursive coordinate bisection (MeshPartition)
# ---------------------------------------------------------------------------

def _perm_box(cells, seed=0):
    g = tb.generate_box_mesh(*cells)
    return tb.permute_nodes(g, np.random.default_rng(seed).permutation(g.n_nodes))


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_rcb_parts_balanced_and_deterministic(world):
    from paper_2403_08777_b200.distributed import rcb_parts
    m = _perm_box((6, 5, 4))
    cen = m.coords[m.connectivity].mean(axis=1)
    p = rcb_parts(cen, world)
    assert p.shape == (m.n_elems,) and p.min() == 0 and p.max() == world - 1
    counts = np.bincount(p, minlength=world)
    assert counts.max() - counts.min() <= np.ceil(np.log2(max(world, 2)))  # one per bisection level
    np.testing.assert_array_equal(p, rcb_parts(cen, world))


@pytest.mark.parametrize("world", [2, 3, 4, 7])
def test_mesh_partition_invariants(world):
    from paper_2403_08777_b200.distributed import MeshPartition
    m = _perm_box((5, 4, 6), seed=1)
    parts = [MeshPartition(m, r, world) for r in range(world)]
    # every element exactly once, local meshes are re-indexed slices
    elems = np.sort(np.concatenate([p.elements for p in parts]))
    np.testing.assert_array_equal(elems, np.arange(m.n_elems))
    owned = np.zeros(m.n_nodes, dtype=int)
    for p in parts:
        lm = p.local_mesh()
        np.testing.assert_array_equal(p.global_nodes[lm.connectivity], m.connectivity[p.elements])
        np.testing.assert_array_equal(lm.coords, m.coords[p.global_nodes])
        owned[p.global_nodes[p.owned_mask()]] += 1
        for nbr, ids in p.interfaces().items():
            q = parts[nbr]
            other = q.interfaces()[p.rank]
            np.testing.assert_array_equal(p.global_nodes[ids], q.global_nodes[other])
    assert (owned == 1).all()  # each global node reported by exactly one rank


def _worker_rcb(rank, world, port, cells, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2403_08777_b200.distributed import MeshPartition
    g = _perm_box(cells, seed=2)
    p = MeshPartition(g, rank, world)
    m = p.local_mesh()
    u = p.velocity(tb.make_velocity(g, "random:1"))
    rhs = O.assemble_rsp(m.coords, m.connectivity, u)  # stand-in for the GPU local assembly
    send = {n: torch.from_numpy(rhs[ids].copy()) for n, ids in p.interfaces().items()}
    recv = {n: torch.empty_like(t) for n, t in send.items()}
    exchange_interfaces(p, send, recv)
    for nbr, ids in p.interfaces().items():
        rhs[ids] += recv[nbr].numpy()
    np.save(os.path.join(out_dir, f"rhs_{rank}.npy"), rhs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [3, 4])
def test_rcb_exchange_gloo_matches_single_domain(tmp_path, world, oracle):
    """Nodes shared by up to 4 ranks and ranks with several neighbours: the
    pairwise exchange of local partials still gives every sharer the sum."""
    from paper_2403_08777_b200.distributed import MeshPartition
    cells = (5, 4, 6)
    mp.start_processes(_worker_rcb, args=(world, _free_port(), cells, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    g = _perm_box(cells, seed=2)
    ug = tb.make_velocity(g, "random:1")
    ref = oracle.assemble_rsp(g.coords, g.connectivity, ug)
    full = np.full_like(ref, np.nan)
    nbrs = 0
    for r in range(world):
        p = MeshPartition(g, r, world)
        loc = np.load(tmp_path / f"rhs_{r}.npy")
        full[p.global_nodes[p.owned_mask()]] = loc[p.owned_mask()]
        ref_loc = ref[p.global_nodes]
        assert np.abs(loc - ref_loc).max() <= 1e-12 * np.abs(ref).max()  # every sharer has the sum
        nbrs = max(nbrs, len(p.interfaces()))
    assert nbrs >= 2
    assert not np.isnan(full).any()
    assert oracle.compare(full, ref, g.coords, g.connectivity, ug).passed


def _rcb_numpy(points, world):
    """The numpy statement of RCB (round 1's implementation, kept here as the
    checker of the native partitioner)."""
    pts = np.asarray(points, dtype=np.float64)
    part = np.zeros(pts.shape[0], dtype=np.int32)
    stack = [(np.arange(pts.shape[0]), 0, world)]
    while stack:
        idx, first, k = stack.pop()
        if k == 1 or idx.size == 0:
            part[idx] = first
            continue
        kl = k // 2
        sub = pts[idx]
        ax = int(np.argmax(sub.max(axis=0) - sub.min(axis=0)))
        order = np.argsort(sub[:, ax], kind="stable")
        cut = (idx.size * kl) // k
        stack.append((idx[order[:cut]], first, kl))
        stack.append((idx[order[cut:]], first + kl, k - kl))
    return part


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 7, 8, 16])
@pytest.mark.parametrize("case", ["box", "permuted", "ties", "random"])
def test_native_rcb_equals_numpy_statement(world, case):
    from paper_2403_08777_b200.distributed import rcb_parts
    if case == "box":
        m = tb.generate_box_mesh(9, 7, 5)
        pts = m.coords[m.connectivity].mean(axis=1)
    elif case == "permuted":
        m = _perm_box((8, 6, 7), seed=3)
        pts = m.coords[m.connectivity].mean(axis=1)
    elif case == "ties":  # many equal coordinates: the stable order decides
        pts = np.floor(np.random.default_rng(1).uniform(0, 4, (3000, 3)))
    else:
        pts = np.random.default_rng(2).normal(size=(20000, 3)) * [1.0, 3.0, 0.5]
    np.testing.assert_array_equal(rcb_parts(pts, world), _rcb_numpy(pts, world))

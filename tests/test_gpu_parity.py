"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle and
the reference's golden vectors.  Run on a B200 with ``pytest -m gpu``.

Criteria (oracle.compare): the reference's max|d|/denominator <= 1e-12
(variants.py:62-65, 653-711) AND north_star's rel-L2 <= 1e-12 and
max|d| <= 1e-10 * ||oracle||_inf.  Atomic scatter is compared with these
tolerances; 'private' and 'colored' must additionally rerun bitwise.
"""
import numpy as np
import pytest

import paper_2403_08777_b200 as tb
from conftest import INITS, SMALL_DIMS, dims_key, init_key

pytestmark = pytest.mark.gpu

MODES = ["private", "private-atomic", "atomic", "colored"]
P = tb.PhysParams()


def run(mesh, u, params=P, **cfg):
    return tb.assemble_rsp(mesh, u, params, tb.RunConfig(**cfg))


def assert_parity(oracle, rhs, ref, mesh, u, params=P):
    chk = oracle.compare(rhs, ref, mesh.coords, mesh.connectivity, u, params.rho, params.mu,
                         params.c_vreman)
    assert chk.passed, chk
    return chk


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("init", INITS)
@pytest.mark.parametrize("dims", SMALL_DIMS)
def test_small_boxes_against_reference_goldens(oracle, golden_small, dims, init, mode):
    m = tb.generate_box_mesh(*dims)
    k, ik = dims_key(dims), init_key(init)
    u = golden_small[f"u_{k}_{ik}"]
    res = run(m, u, scatter=mode)
    assert_parity(oracle, res.rhs, golden_small[f"oracle_{k}_{ik}"], m, u)
    assert_parity(oracle, res.rhs, golden_small[f"rsp_{k}_{ik}"], m, u)


@pytest.mark.parametrize("renumber", ["none", "rcm", "sfc"])
@pytest.mark.parametrize("order", ["keep", "node", "sfc"])
def test_renumbering_and_element_order(oracle, golden_mid, renumber, order):
    m = tb.generate_box_mesh(8, 8, 8)
    u = tb.make_velocity(m, "random:1")
    for mode in MODES:
        res = run(m, u, scatter=mode, renumber=renumber, element_order=order)
        assert_parity(oracle, res.rhs, golden_mid["oracle_8_random"], m, u)


@pytest.mark.parametrize("patches", ["star", "tet"])
@pytest.mark.parametrize("cp,cn", [(1, 16), (7, 16), (64, 144), (64, 40), (100, 256), (128, 256),
                                   (128, 64), (128, 16)])
def test_chunk_shape_invariance(oracle, golden_mid, patches, cp, cn):
    m = tb.generate_box_mesh(16, 16, 16)
    u = tb.make_velocity(m, "taylor-green")
    ref = golden_mid["rsp_16_taylor-green"]
    for mode in ("private", "private-atomic"):
        res = run(m, u, scatter=mode, patches=patches, cta_patches=cp, chunk_nodes=cn)
        assert_parity(oracle, res.rhs, ref, m, u)


def test_mid_size_goldens(oracle, golden_mid):
    for n in (8, 16):
        m = tb.generate_box_mesh(n, n, n)
        for init in ("random:1", "taylor-green"):
            u = tb.make_velocity(m, init)
            for mode in MODES:
                rhs = run(m, u, scatter=mode).rhs
                assert_parity(oracle, rhs, golden_mid[f"rsp_{n}_{init_key(init)}"], m, u)


def test_32cubed_checksums(oracle, golden_checksums):
    m = tb.generate_box_mesh(32, 32, 32)
    for init in ("taylor-green", "random:1"):
        u = tb.make_velocity(m, init)
        ref = oracle.assemble_rsp(m.coords, m.connectivity, u, n_threads=oracle.default_threads())
        s, sa, mx = golden_checksums[f"sum_32_{init_key(init)}"]
        for mode in MODES:
            rhs = run(m, u, scatter=mode).rhs
            assert_parity(oracle, rhs, ref, m, u)
            assert abs(np.abs(rhs).sum() - sa) <= 1e-12 * sa
            assert abs(np.abs(rhs).max() - mx) <= 1e-12 * mx


@pytest.mark.parametrize("mode", ["private", "colored"])
def test_bitwise_reruns(mode):
    m = tb.generate_box_mesh(12, 10, 9)
    u = tb.make_velocity(m, "random:3")
    a = run(m, u, scatter=mode).rhs
    for _ in range(3):
        np.testing.assert_array_equal(run(m, u, scatter=mode).rhs, a)


def test_modes_agree():
    m = tb.generate_box_mesh(10, 11, 12)
    u = tb.make_velocity(m, "random:7")
    base = run(m, u, scatter="private").rhs
    scale = np.abs(base).max()
    for mode in MODES[1:]:
        assert np.abs(run(m, u, scatter=mode).rhs - base).max() <= 1e-12 * scale


def test_reference_tet_single_element(oracle, golden_small):
    m = tb.Mesh(coords=golden_small["reftet_coords"], connectivity=golden_small["reftet_conn"])
    u = golden_small["reftet_u"]
    for mode in MODES:
        rhs = run(m, u, scatter=mode).rhs
        assert_parity(oracle, rhs, golden_small["reftet_oracle"], m, u)


def test_linear_field_analytic(golden_small):
    """u=(x,0,0), rho=mu=1, c=0 on the reference tet (test_kernel.py:205-223)."""
    m = tb.Mesh(coords=golden_small["reftet_coords"], connectivity=golden_small["reftet_conn"])
    p = tb.PhysParams(rho=1.0, mu=1.0, c_vreman=0.0)
    rhs = run(m, golden_small["reftet_linx_u"], p).rhs
    np.testing.assert_allclose(rhs, golden_small["reftet_linx_oracle"], rtol=1e-13, atol=1e-18)


def test_nondefault_physics(oracle, golden_small):
    m = tb.generate_box_mesh(3, 3, 3)
    rho, mu, cv = golden_small["phys_params"]
    p = tb.PhysParams(rho=float(rho), mu=float(mu), c_vreman=float(cv))
    u = golden_small["phys_u"]
    for mode in MODES:
        assert_parity(oracle, run(m, u, p, scatter=mode).rhs, golden_small["phys_oracle"], m, u, p)


def test_permuted_numbering(oracle, golden_small):
    m = tb.Mesh(coords=golden_small["perm6_coords"], connectivity=golden_small["perm6_conn"])
    u = golden_small["perm6_u"]
    for renumber in ("none", "rcm", "sfc"):
        rhs = run(m, u, renumber=renumber).rhs
        assert_parity(oracle, rhs, golden_small["perm6_oracle"], m, u)


def test_translation_invariance(golden_small):
    m = tb.generate_box_mesh(3, 3, 3)
    sh = tb.Mesh(coords=m.coords + np.array([10.0, -20.0, 5.0]), connectivity=m.connectivity)
    u = golden_small["shift_u"]
    a, b = run(m, u).rhs, run(sh, u).rhs
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()


def test_zero_and_constant_fields_exact():
    m = tb.generate_box_mesh(4, 3, 5)
    for spec in ("zero", "constant:0.9,0.1,-0.4"):
        u = tb.make_velocity(m, spec)
        for mode in MODES:
            np.testing.assert_array_equal(run(m, u, scatter=mode).rhs, np.zeros((m.n_nodes, 3)))


def test_shear_field_has_no_eddy_viscosity():
    """Rank-1 gradient -> nu_t = 0 exactly (kernel.py:104-111): c_vreman is inert."""
    m = tb.generate_box_mesh(5, 5, 5)
    u = tb.make_velocity(m, "shear:1.5")
    a = run(m, u, tb.PhysParams(c_vreman=0.07), scatter="private").rhs
    b = run(m, u, tb.PhysParams(c_vreman=0.0), scatter="private").rhs
    np.testing.assert_array_equal(a, b)


def test_empty_mesh():
    m = tb.Mesh(coords=np.array([[0.0, 0, 0], [1.0, 0, 0]]), connectivity=np.zeros((0, 4), np.int64))
    for mode in MODES:
        np.testing.assert_array_equal(run(m, np.zeros((2, 3)), scatter=mode).rhs, np.zeros((2, 3)))


def test_isolated_nodes_are_zero(oracle):
    """A node no element touches gets 0 in every mode (private merge writes it)."""
    base = tb.generate_box_mesh(3, 3, 3)
    coords = np.vstack([base.coords, [[5.0, 5.0, 5.0]]])
    m = tb.Mesh(coords=coords, connectivity=base.connectivity)
    u = np.random.default_rng(0).uniform(-1, 1, (m.n_nodes, 3))
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u)
    for mode in MODES:
        rhs = run(m, u, scatter=mode).rhs
        assert np.all(rhs[-1] == 0.0)
        assert_parity(oracle, rhs, ref, m, u)


def test_precolored_mesh(oracle):
    m = tb.color_elements(tb.generate_box_mesh(4, 4, 4))
    u = tb.make_velocity(m, "random:2")
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u)
    assert_parity(oracle, run(m, u, scatter="colored").rhs, ref, m, u)


def test_general_pmat_kernel(oracle):
    """A non-symmetric interpolation table takes the general-moment kernel."""
    m = tb.generate_box_mesh(4, 3, 3)
    u = tb.make_velocity(m, "random:5")
    pm = np.random.default_rng(3).uniform(0.0, 0.5, (4, 4))
    ids = np.arange(m.n_elems, dtype=np.int64)
    ref = np.zeros((m.n_nodes, 3))
    oracle.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids, ref)
    asm = tb.Assembler(m, tb.RunConfig(), build_colors=True)
    for scatter in ("private-atomic", "atomic", "colored"):
        rhs = np.empty((m.n_nodes, 3))
        asm.assemble_into(u, P, rhs, scatter, pmat=pm)
        assert_parity(oracle, rhs, ref, m, u)
    # 'private' promises a bitwise reproducible sum: refused, not silently atomic
    with pytest.raises(ValueError, match="symmetric"):
        asm.assemble_into(u, P, np.empty((m.n_nodes, 3)), "private", pmat=pm)
    asm.close()


def test_assemble_elements_seam_accumulates(oracle):
    """Mirror of _rsp_kernels.assemble_elements: subset ids, += into rhs."""
    m = tb.generate_box_mesh(4, 4, 3)
    u = tb.make_velocity(m, "random:8")
    pm = tb.interpolation_table()
    ids = np.arange(1, m.n_elems, 3, dtype=np.int64)
    start = np.random.default_rng(1).uniform(-1, 1, (m.n_nodes, 3))
    ref = start.copy()
    oracle.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids, ref)
    got = start.copy()
    tb.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids, got)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    with pytest.raises(ValueError):
        tb.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm,
                             np.array([m.n_elems]), got)


def test_device_resident_path_and_torch_views(oracle):
    import torch
    m = tb.generate_box_mesh(9, 8, 7)
    u = tb.make_velocity(m, "random:4")
    asm = tb.Assembler(m, tb.RunConfig())
    rhs_host, _ = asm.assemble(u, P)
    asm.set_velocity_host(u)
    nl = asm.run(P)
    assert nl >= 1
    out = asm.get_rhs_host()
    asm.synchronize()
    np.testing.assert_array_equal(out, rhs_host)
    views = asm.torch_views()
    perm = np.arange(m.n_nodes) if asm.device_buffers()["perm"] is None else None
    rx = views["rx"].cpu().numpy()
    ids = asm.map_nodes(np.arange(m.n_nodes))
    np.testing.assert_array_equal(rx[ids], rhs_host[:, 0])
    assert perm is None or perm.size == m.n_nodes
    # velocity written through the torch view drives the next run
    views["ux"].zero_(); views["uy"].zero_(); views["uz"].zero_()
    torch.cuda.synchronize()
    asm.run(P)
    np.testing.assert_array_equal(asm.get_rhs_host(), np.zeros((m.n_nodes, 3)))
    asm.close()


def test_result_fields():
    m = tb.generate_box_mesh(2, 2, 2)
    u = tb.make_velocity(m, "random:1")
    res = run(m, u)
    assert res.variant is tb.VariantId.RSP and res.wall_time > 0.0
    assert res.elements_per_second == pytest.approx(m.n_elems / res.wall_time, rel=1e-9)
    assert np.isfinite(res.rhs).all()
    assert res.timings.kernel_launches >= 1


def test_velocity_validation_on_gpu_path():
    m = tb.generate_box_mesh(2, 2, 2)
    u = np.zeros((m.n_nodes, 3))
    u[3, 1] = np.nan
    with pytest.raises(ValueError):
        run(m, u)
    with pytest.raises(ValueError):
        run(m, np.zeros((3, m.n_nodes)))


@pytest.mark.parametrize("init", ["random:1", "taylor-green"])
def test_full_size_128(oracle, init):
    """BASELINE config 2 at full size: 128^3 (12.58M tets), all modes,
    against the threaded C oracle (same arithmetic as the reference)."""
    m = tb.generate_box_mesh(128, 128, 128)
    u = tb.make_velocity(m, init)
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u, n_threads=oracle.default_threads(),
                              vector_dim=4096)
    for mode in ("private", "private-atomic", "atomic"):
        rhs = run(m, u, scatter=mode).rhs
        assert_parity(oracle, rhs, ref, m, u)
    tb.clear_cache()


def test_full_size_128_random_permutation(oracle):
    """BASELINE config 3: 128^3 with randomly permuted node numbering."""
    base = tb.generate_box_mesh(128, 128, 128)
    perm = np.random.default_rng(0).permutation(base.n_nodes)
    m = tb.permute_nodes(base, perm)
    u = tb.make_velocity(m, "random:1")
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u, n_threads=oracle.default_threads(),
                              vector_dim=4096)
    for renumber in ("none", "rcm"):
        rhs = run(m, u, renumber=renumber, element_order="keep" if renumber == "none" else "sfc").rhs
        assert_parity(oracle, rhs, ref, m, u)
    tb.clear_cache()


def test_async_pipeline_matches_sync():
    """tal_assemble_async: several fields in flight give the same results as
    the blocking call (pinned and pageable host buffers)."""
    from paper_2403_08777_b200._native import PinnedArray
    m = tb.generate_box_mesh(14, 12, 10)
    asm = tb.Assembler(m, tb.RunConfig())
    fields = [tb.make_velocity(m, f"random:{s}") for s in range(7)]
    ref = [asm.assemble(f, P)[0] for f in fields]
    pins = [PinnedArray((m.n_nodes, 3)) for _ in range(4)]
    for k, f in enumerate(fields[:2]):
        pins[k].array[:] = f
    outs = [np.empty((m.n_nodes, 3)) for _ in fields]
    tickets = []
    for k, f in enumerate(fields):
        src = pins[k].array if k < 2 else f
        tickets.append(asm.assemble_async(src, P, outs[k]))
    for t in tickets:
        asm.wait(t)
    for k in range(len(fields)):
        np.testing.assert_array_equal(outs[k], ref[k])
    for p_ in pins:
        p_.free()
    asm.close()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_domains_loopback_on_one_gpu(oracle, world):
    """The multi-GPU decomposition on one device: each slab assembled by its
    own Assembler (RCM-renumbered), interface planes exchanged by device
    copies standing in for the NCCL send/recv, accumulated by the halo
    kernels; the owned rows reproduce the single-domain oracle."""
    import torch
    from paper_2403_08777_b200.distributed import SlabPartition
    cells = (9, 8, 12)
    parts = [SlabPartition(cells, r, world) for r in range(world)]
    doms = []
    for p in parts:
        m = p.local_mesh()
        asm = tb.Assembler(m, tb.RunConfig(scatter="private-atomic"))
        asm.set_velocity_host(p.velocity("random:1", m), stream=0)
        doms.append((p, m, asm))
    for p, m, asm in doms:
        asm.run(P, stream=0)
    bufs = {}
    for p, m, asm in doms:
        for nbr, ids in p.interfaces().items():
            lst = torch.as_tensor(asm.map_nodes(ids), device="cuda")
            out = torch.empty((ids.size, 3), dtype=torch.float64, device="cuda")
            asm.halo_pack(lst.data_ptr(), lst.numel(), out.data_ptr(), stream=0)
            bufs[(p.rank, nbr)] = (lst, out)
    for p, m, asm in doms:
        for nbr in p.interfaces():
            lst, _ = bufs[(p.rank, nbr)]
            _, recv = bufs[(nbr, p.rank)]
            asm.halo_accumulate(lst.data_ptr(), lst.numel(), recv.data_ptr(), stream=0)
    torch.cuda.synchronize()
    g = oracle.box_mesh(*cells)
    ug = oracle.velocity(g.coords, "random:1")
    ref = oracle.assemble_rsp(g.coords, g.connectivity, ug)
    full = np.full_like(ref, np.nan)
    for p, m, asm in doms:
        lo, hi = p.node_range
        loc = asm.get_rhs_host(stream=0)
        asm.synchronize(stream=0)
        mask = p.owned_mask()
        full[lo:hi][mask] = loc[mask]
        asm.close()
    assert not np.isnan(full).any()
    assert_parity(oracle, full, ref, g, ug)


def test_extreme_scales_all_modes(oracle):
    """Tiny and huge mesh/velocity scales, non-default physics: every scatter
    mode within tolerance, the deterministic ones bitwise reproducible."""
    for ext, amp in [((1e-6, 1e-6, 1e-6), 1e3), ((1e3, 2e3, 5e2), 1e-4), ((1.0, 1.0, 1.0), 1e8)]:
        m = tb.generate_box_mesh(7, 6, 5, extents=ext)
        u = amp * np.random.default_rng(9).uniform(-1, 1, (m.n_nodes, 3))
        p = tb.PhysParams(rho=2.0, mu=3e-3, c_vreman=0.1)
        ref = oracle.assemble_rsp(m.coords, m.connectivity, u, p.rho, p.mu, p.c_vreman)
        for mode in MODES:
            a = run(m, u, p, scatter=mode).rhs
            assert_parity(oracle, a, ref, m, u, p)
            if mode in ("private", "colored"):
                np.testing.assert_array_equal(a, run(m, u, p, scatter=mode).rhs)


@pytest.mark.parametrize("world", [2, 3])
def test_fused_interface_sum_in_process(oracle, world):
    """Fused interface sum: each slab's kernel REDs its interface partials into
    the neighbour's RHS through peer pointers (here in-process, one device),
    ordered by the device flag words; owned rows match the single-domain oracle,
    and repeated steps (epochs) stay correct."""
    from paper_2403_08777_b200.distributed import SlabPartition
    cells = (8, 7, 10)
    doms = []
    for r in range(world):
        p = SlabPartition(cells, r, world)
        m = p.local_mesh()
        ext = np.concatenate(list(p.interfaces().values()))
        asm = tb.Assembler(m, tb.RunConfig(scatter="private-atomic"), external_nodes=ext)
        asm.set_velocity_host(p.velocity("random:1", m))
        doms.append((p, m, asm))
    for p, m, asm in doms:
        for nbr, ids in p.interfaces().items():
            q, _, asq = doms[nbr]
            rx, fl, n = asq.peer_local()
            slot = 0 if nbr < p.rank else 1
            asm.peer_attach(slot, rx, n, fl, ids, asq.map_nodes(q.interfaces()[p.rank]))
    g = oracle.box_mesh(*cells)
    ug = oracle.velocity(g.coords, "random:1")
    ref = oracle.assemble_rsp(g.coords, g.connectivity, ug)
    for step in range(5):
        if step == 3:  # then as captured CUDA graphs (device-side flag epochs)
            for p, m, asm in doms:
                asm.capture(P)
        for p, m, asm in doms:
            if step < 3:
                asm.run(P)  # internal streams: the ranks' flag waits overlap
            else:
                asm.replay()
        full = np.full_like(ref, np.nan)
        for p, m, asm in doms:
            loc = asm.get_rhs_host()
            asm.synchronize()
            lo, hi = p.node_range
            mask = p.owned_mask()
            full[lo:hi][mask] = loc[mask]
            for nbr, ids in p.interfaces().items():  # both copies of a plane agree
                assert np.abs(loc[ids]).max() > 0
        assert not np.isnan(full).any()
        assert_parity(oracle, full, ref, g, ug)
    for _, _, asm in doms:
        asm.peer_detach()
        asm.close()


@pytest.mark.parametrize("world", [3, 5])
def test_rcb_partitions_loopback_on_one_gpu(oracle, world):
    """General-mesh decomposition (RCB of a randomly renumbered box): every
    part assembled by its own Assembler, the shared-node partials of all
    neighbour pairs exchanged by device copies standing in for NCCL, the
    owned rows reproduce the single-domain oracle."""
    import torch
    from paper_2403_08777_b200.distributed import MeshPartition
    g = tb.generate_box_mesh(10, 9, 8)
    g = tb.permute_nodes(g, np.random.default_rng(7).permutation(g.n_nodes))
    ug = tb.make_velocity(g, "random:1")
    doms = []
    for r in range(world):
        p = MeshPartition(g, r, world)
        asm = tb.Assembler(p.local_mesh(), tb.RunConfig(scatter="private-atomic"))
        asm.set_velocity_host(p.velocity(ug), stream=0)
        asm.run(P, stream=0)
        doms.append((p, asm))
    bufs = {}
    for p, asm in doms:  # every local partial packed before any accumulation
        for nbr, ids in p.interfaces().items():
            lst = torch.as_tensor(asm.map_nodes(ids), device="cuda")
            out = torch.empty((ids.size, 3), dtype=torch.float64, device="cuda")
            asm.halo_pack(lst.data_ptr(), lst.numel(), out.data_ptr(), stream=0)
            bufs[(p.rank, nbr)] = (lst, out)
    for p, asm in doms:
        for nbr in p.interfaces():
            lst, _ = bufs[(p.rank, nbr)]
            asm.halo_accumulate(lst.data_ptr(), lst.numel(), bufs[(nbr, p.rank)][1].data_ptr(),
                                stream=0)
    torch.cuda.synchronize()
    ref = oracle.assemble_rsp(g.coords, g.connectivity, ug)
    full = np.full_like(ref, np.nan)
    for p, asm in doms:
        loc = asm.get_rhs_host(stream=0)
        asm.synchronize(stream=0)
        full[p.global_nodes[p.owned_mask()]] = loc[p.owned_mask()]
        asm.close()
    assert not np.isnan(full).any()
    assert_parity(oracle, full, ref, g, ug)


def test_cuda_graph_replay_matches_run(oracle):
    """tal_graph_capture/launch: one captured step replays the assembly on the
    handle's buffers -- bitwise equal to run() for 'private', picks up new
    velocity and pressure contents, refuses handles with peers."""
    import torch
    m = tb.generate_box_mesh(12, 10, 9)
    fields = [tb.make_velocity(m, f"random:{s}") for s in (1, 2)]
    for scatter in ("private", "private-atomic", "atomic", "colored"):
        asm = tb.Assembler(m, tb.RunConfig(scatter=scatter))
        asm.set_velocity_host(fields[0], stream=0)
        asm.run(P, stream=0)
        ref = asm.get_rhs_host(stream=0)
        asm.synchronize(stream=0)
        asm.capture(P)
        for u in fields:
            asm.set_velocity_host(u, stream=0)
            n = asm.replay(stream=0)
            got = asm.get_rhs_host(stream=0)
            asm.synchronize(stream=0)
            assert n >= 1
            want = oracle.assemble_rsp(m.coords, m.connectivity, u)
            assert_parity(oracle, got, want, m, u)
        asm.set_velocity_host(fields[0], stream=0)
        asm.replay(stream=0)
        again = asm.get_rhs_host(stream=0)
        asm.synchronize(stream=0)
        if scatter in ("private", "colored"):
            np.testing.assert_array_equal(again, ref)
        asm.close()
    # pressure captured with the graph
    p = np.random.default_rng(1).uniform(-1, 1, m.n_nodes)
    asm = tb.Assembler(m, tb.RunConfig(scatter="private-atomic"))
    asm.set_pressure(p)
    asm.set_velocity_host(fields[1], stream=0)
    asm.capture(P)
    asm.replay(stream=torch.cuda.current_stream())
    got = asm.get_rhs_host(stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    want = oracle.assemble_rsp(m.coords, m.connectivity, fields[1]) + \
        oracle.pressure_gradient(m.coords, m.connectivity, p)
    assert_parity(oracle, got, want, m, fields[1])
    asm.close()


def test_bad_colour_ids_are_rejected():
    """Negative or huge colour ids pass the (node, colour) uniqueness check
    but index per-colour tables: refused with ValueError at upload."""
    m = tb.generate_box_mesh(2, 2, 2)
    for bad in (-1, m.n_elems, 1 << 40):
        cols = np.arange(m.n_elems, dtype=np.int64)
        cols[3] = bad
        mc = tb.Mesh(coords=m.coords, connectivity=m.connectivity, colors=cols)
        with pytest.raises(ValueError, match="colour ids"):
            tb.Assembler(mc, tb.RunConfig(scatter="colored"))


@pytest.mark.parametrize("which", ["all", "range", "slabs", "scattered", "repeated"])
@pytest.mark.parametrize("general", [False, True])
def test_fast_seam_paths(oracle, which, general):
    """tal_seam_*: the whole mesh (edge-star kernel), a contiguous range and
    thread slabs (per-element kernel over the resident conn), an arbitrary
    and a repeated id list (uploaded ids) -- each accumulating into rhs like
    the numba loop, for the symmetric and a general pmat."""
    m = tb.generate_box_mesh(7, 6, 5)
    u = tb.make_velocity(m, "random:12")
    pm = np.random.default_rng(4).uniform(0.0, 0.5, (4, 4)) if general else tb.interpolation_table()
    E = m.n_elems
    groups = {"all": [np.arange(E)], "range": [np.arange(17, 433)],
              "slabs": [np.arange(lo, min(lo + 160, E)) for lo in range(0, E, 160)],
              "scattered": [np.random.default_rng(2).permutation(E)[: E // 3]],
              "repeated": [np.array([5, 5, 9, 0, 5, E - 1])]}[which]
    start = np.random.default_rng(1).uniform(-1, 1, (m.n_nodes, 3))
    ref, got = start.copy(), start.copy()
    for ids in groups:
        ids = ids.astype(np.int64)
        oracle.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids, ref)
        tb.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids, got)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_stateless_seam_entry_sees_changed_arrays(oracle):
    """tal_assemble_elements (the plain C entry) caches the resident mesh by
    address + content hash: an in-place change of coords is re-uploaded."""
    import ctypes
    from paper_2403_08777_b200 import _native as N
    m = tb.generate_box_mesh(5, 4, 4)
    coords = np.array(m.coords)
    conn = np.array(m.connectivity)
    u = tb.make_velocity(m, "random:3")
    pm = tb.interpolation_table()
    ids = np.arange(m.n_elems, dtype=np.int64)

    def call():
        out = np.zeros((m.n_nodes, 3))
        N.check(N.lib().tal_assemble_elements(0, N.ptr(coords), N.ptr(conn), coords.shape[0],
                                              conn.shape[0], N.ptr(u), 1.0, 1e-3, 0.07, N.ptr(pm),
                                              N.ptr(ids), ids.shape[0], N.ptr(out)))
        ref = np.zeros_like(out)
        oracle.assemble_elements(coords, conn, u, 1.0, 1e-3, 0.07, pm, ids, ref)
        assert np.abs(out - ref).max() <= 1e-13 * np.abs(ref).max()
        return out

    a = call()
    b = call()  # cached context
    assert np.array_equal(a, b) or np.abs(a - b).max() <= 1e-15 * np.abs(a).max()
    coords *= 1.5  # same address, new content
    c = call()
    assert not np.allclose(a, c)
    del ctypes


def test_stateless_seam_range_calls_see_changes_they_read(oracle):
    """Slab calls on the stateless entry check the fingerprints of the blocks
    they read (their conn rows and coords rows): a change inside a later
    slab's rows, or of connectivity, is re-uploaded before that slab runs."""
    from paper_2403_08777_b200 import _native as N
    m = tb.generate_box_mesh(40, 30, 30)  # coords 0.9 MB, conn 4.6 MB: many fingerprint blocks
    coords = np.array(m.coords)
    conn = np.array(m.connectivity)
    u = tb.make_velocity(m, "random:3")
    pm = tb.interpolation_table()
    E = m.n_elems

    def call(ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.zeros((m.n_nodes, 3))
        N.check(N.lib().tal_assemble_elements(0, N.ptr(coords), N.ptr(conn), coords.shape[0],
                                              conn.shape[0], N.ptr(u), 1.0, 1e-3, 0.07, N.ptr(pm),
                                              N.ptr(ids), ids.shape[0], N.ptr(out)))
        ref = np.zeros_like(out)
        oracle.assemble_elements(coords, conn, u, 1.0, 1e-3, 0.07, pm, ids, ref)
        assert np.abs(out - ref).max() <= 1e-13 * np.abs(ref).max()
        return out

    lo, hi = np.arange(0, E // 4), np.arange(3 * E // 4, E)
    call(lo)
    call(hi)
    v = int(conn[hi[-1], 0])
    coords[v] += 0.01  # a node only the last slab reads
    call(lo)
    call(hi)
    conn[hi[10], [1, 2]] = conn[hi[10], [2, 1]]  # connectivity change (orientation flip)
    call(hi)
    call(np.arange(E))


def test_fast_seam_from_a_thread_pool(oracle):
    """The reference's threaded private driver (variants.py:578-596): slab
    calls from a ThreadPoolExecutor, one accumulator per thread, merged in
    thread order -- the fast seam under concurrency (serialised GPU part,
    per-call node-row windows)."""
    from concurrent.futures import ThreadPoolExecutor
    m = tb.generate_box_mesh(24, 20, 18)
    u = tb.make_velocity(m, "random:5")
    pm = tb.interpolation_table()
    E, T = m.n_elems, 8
    ids = np.arange(E, dtype=np.int64)
    cut = [E * t // T for t in range(T + 1)]
    bufs = [np.zeros((m.n_nodes, 3)) for _ in range(T)]
    for _ in range(2):
        for b in bufs:
            b[:] = 0.0
        with ThreadPoolExecutor(T) as pool:
            fs = [pool.submit(tb.assemble_elements, m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm,
                              ids[cut[t]:cut[t + 1]], bufs[t]) for t in range(T)]
            for f in fs:
                f.result()
        got = bufs[0].copy()
        for b in bufs[1:]:
            got += b
        ref = oracle.assemble_rsp(m.coords, m.connectivity, u)
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("renumber", ["rcm", "sfc", "none"])
@pytest.mark.parametrize("permuted", [False, True])
def test_run_caller_fused_layout(oracle, renumber, permuted):
    """tal_run_caller: u read from / rhs written to the caller's own (N,3)
    device arrays by the private kernel (no pack/unpack).  'private' is
    bitwise the internal-layout result; every mode matches the oracle."""
    import torch
    g = tb.generate_box_mesh(10, 9, 8)
    m = tb.permute_nodes(g, np.random.default_rng(5).permutation(g.n_nodes)) if permuted else g
    u = tb.make_velocity(m, "random:9")
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u)
    asm = tb.Assembler(m, tb.RunConfig(renumber=renumber), build_colors=True)
    d_u = torch.as_tensor(u, device="cuda:0").contiguous()
    for scatter in ("private", "private-atomic", "atomic", "colored"):
        d_r = torch.full_like(d_u, float("nan"))
        nl = asm.run_caller(P, d_u.data_ptr(), d_r.data_ptr(), scatter=scatter, stream=0)
        torch.cuda.synchronize()
        got = d_r.cpu().numpy()
        assert_parity(oracle, got, ref, m, u)
        if scatter == "private":
            host, _ = asm.assemble(u, P, scatter="private")
            np.testing.assert_array_equal(got, host)
            assert nl <= 2  # kernel (+ ordered merge): no pack/unpack
    asm.set_pressure(np.zeros(m.n_nodes))  # not fused: the composition path, same numbers
    d_r = torch.empty_like(d_u)
    asm.run_caller(P, d_u.data_ptr(), d_r.data_ptr(), scatter="private", stream=0)
    torch.cuda.synchronize()
    assert_parity(oracle, d_r.cpu().numpy(), ref, m, u)
    asm.close()


@pytest.fixture(scope="module")
def delaunay_mesh():
    return tb.generate_delaunay_mesh(20000, seed=5)  # ~130 K tets, irregular rings


@pytest.mark.parametrize("scatter", ["private", "private-atomic", "atomic", "colored", "sequential"])
def test_unstructured_delaunay_mesh(oracle, delaunay_mesh, scatter):
    """A genuinely unstructured mesh (Delaunay of random points: open and
    closed edge rings of every size, irregular valences) in every scatter
    mode, against the oracle on the same arrays."""
    m = delaunay_mesh
    u = tb.make_velocity(m, "random:6")
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u)
    res = tb.assemble_rsp(m, u, tb.PhysParams(), tb.RunConfig(scatter=scatter))
    chk = oracle.compare(res.rhs, ref, m.coords, m.connectivity, u)
    assert chk.passed, chk


def test_unstructured_delaunay_mesh_layouts(oracle, delaunay_mesh):
    """Every renumbering x element order on the unstructured mesh, and the
    'private' result bitwise reproducible across reruns."""
    m = delaunay_mesh
    u = tb.make_velocity(m, "taylor-green")
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u)
    for ren in ("rcm", "sfc", "none"):
        for eo in ("sfc", "node", "keep"):
            cfg = tb.RunConfig(scatter="private", renumber=ren, element_order=eo)
            a = tb.assemble_rsp(m, u, tb.PhysParams(), cfg).rhs
            b = tb.assemble_rsp(m, u, tb.PhysParams(), cfg).rhs
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
            assert oracle.compare(a, ref, m.coords, m.connectivity, u).passed, (ren, eo)

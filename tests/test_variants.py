"""The code-shape study: the B, RS and RSP shapes of the
operator on the B200, mirroring the reference's tests/test_variants.py.

CPU tests (no marker): ledgers, the verification arithmetic, and the
reference's own B/RS outputs (tests/golden/rhs_shapes.npz) against the oracle.
GPU tests (@gpu): every shape through the C-ABI against the oracle and the
reference's B/RS vectors, determinism, the verify_variants machinery.
"""
import numpy as np
import pytest

import paper_2403_08777_b200 as tb
from conftest import GOLDEN, INITS, init_key

P = tb.PhysParams()
VARIANTS = list(tb.VariantId)


@pytest.fixture(scope="module")
def golden_shapes():
    return np.load(GOLDEN / "rhs_shapes.npz")


# ---------------------------------------------------------------------------
# CPU: ledgers and comparison arithmetic (variants.py:182-243, 634-711)
# ---------------------------------------------------------------------------

def test_assemblers_cover_every_variant():
    assert set(tb.ASSEMBLERS) == set(tb.VariantId) == {tb.VariantId(v) for v in ("b", "rs", "rsp")}


def test_flop_reduction_ratio_and_monotone_ledgers():
    b, rs, rsp = (tb.VARIANT_INFO[v] for v in (tb.VariantId.B, tb.VariantId.RS, tb.VariantId.RSP))
    assert b.flops_per_elem / rs.flops_per_elem >= 3.0
    assert b.flops_per_elem > rs.flops_per_elem >= rsp.flops_per_elem
    assert b.intermediate_doubles_per_elem > rs.intermediate_doubles_per_elem \
        > rsp.intermediate_doubles_per_elem
    assert b.loadstore_per_elem > rs.loadstore_per_elem > rsp.loadstore_per_elem
    assert rsp.intermediate_arrays == 0 and b.intermediate_arrays >= 3 * rsp.intermediate_arrays
    for v, info in tb.VARIANT_INFO.items():
        assert info.variant is v and info.name and info.flop_formula


def test_dram_model_spills_only_baseline_at_large_chunks():
    small, huge = tb.RunConfig(vector_dim=16), tb.RunConfig(vector_dim=2048 * 1024)
    for v in tb.VariantId:
        assert tb.make_ledger(v, small).bytes_dram_est == 384.0
    assert tb.make_ledger(tb.VariantId.B, huge).bytes_dram_est > 384.0
    assert tb.make_ledger(tb.VariantId.RS, huge).bytes_dram_est == 384.0
    assert tb.make_ledger(tb.VariantId.RSP, huge).bytes_dram_est == 384.0


@pytest.mark.parametrize("init", ["random:1", "constant:0.7,-0.3,0.25", "taylor-green"])
def test_contribution_scale_matches_oracle(oracle, init):
    m = tb.generate_box_mesh(3, 2, 2)
    u = tb.make_velocity(m, init)
    ours = tb.contribution_scale(m, u, P)
    ref = oracle.contribution_scale(m.coords, m.connectivity, u)
    assert ours == pytest.approx(ref, rel=1e-14)
    assert tb.contribution_scale(m, np.zeros((m.n_nodes, 3)), P) == 0.0


def test_nonfinite_output_reports_node(golden_small):
    m = tb.generate_box_mesh(2, 2, 2)
    u = golden_small["u_2x2x2_random"]
    ref = golden_small["oracle_2x2x2_random"]
    rhs = ref.copy()
    rhs[5, 2] = np.inf
    chk = tb.oracle_compare(m, u, P, rhs, tb.VariantId.RS, oracle=ref)
    assert not chk.passed and chk.worst_node == 5 and "non-finite" in chk.note
    chk = tb.oracle_compare(m, u, P, ref, tb.VariantId.RS, oracle=ref)
    assert chk.passed and chk.rel_diff == 0.0


@pytest.mark.parametrize("init", INITS)
@pytest.mark.parametrize("dims", [(2, 2, 2), (3, 2, 1)])
def test_reference_shapes_pin_the_oracle(oracle, golden_small, golden_shapes, dims, init):
    """The reference's own B and RS vectors agree with the oracle restatement
    at the reference tolerance, so they are valid parity targets."""
    k, ik = "x".join(map(str, dims)), init_key(init)
    m = tb.generate_box_mesh(*dims)
    u = golden_small[f"u_{k}_{ik}"]
    ref = oracle.assemble_reference(m.coords, m.connectivity, u)
    for shape in ("b", "rs"):
        chk = oracle.compare(golden_shapes[f"{shape}_{k}_{ik}"], ref, m.coords, m.connectivity, u)
        assert chk.passed, (shape, chk)


# ---------------------------------------------------------------------------
# GPU: every shape through the C-ABI
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("scatter", ["private", "atomic"])
@pytest.mark.parametrize("init", INITS)
@pytest.mark.parametrize("dims", [(2, 2, 2), (3, 2, 1)])
def test_all_variants_match_oracle(oracle, golden_small, golden_shapes, dims, init, scatter):
    k, ik = "x".join(map(str, dims)), init_key(init)
    m = tb.generate_box_mesh(*dims)
    u = golden_small[f"u_{k}_{ik}"]
    ref = golden_small[f"oracle_{k}_{ik}"]
    report = tb.verify_variants(m, u, P, tb.RunConfig(vector_dim=8, scatter=scatter), oracle=ref)
    assert report.passed, report
    assert {c.variant for c in report.checks} == set(tb.VariantId)
    for shape, fn in (("b", tb.assemble_baseline), ("rs", tb.assemble_rs)):
        rhs = fn(m, u, P, tb.RunConfig(scatter=scatter)).rhs
        chk = oracle.compare(rhs, golden_shapes[f"{shape}_{k}_{ik}"], m.coords, m.connectivity, u)
        assert chk.passed, (shape, chk)
        chk = oracle.compare(rhs, ref, m.coords, m.connectivity, u)
        assert chk.passed, (shape, chk)


@pytest.mark.gpu
def test_baseline_taylor_green_box444(oracle, golden_shapes):
    m = tb.generate_box_mesh(4, 4, 4)
    u = tb.make_velocity(m, "taylor-green")
    ref = oracle.assemble_reference(m.coords, m.connectivity, u)
    res = tb.assemble_baseline(m, u, P, tb.RunConfig())
    chk = tb.oracle_compare(m, u, P, res.rhs, tb.VariantId.B, oracle=ref)
    assert chk.passed and chk.rel_diff <= 1e-12, chk
    assert oracle.compare(res.rhs, golden_shapes["b_4x4x4_taylor-green"], m.coords,
                          m.connectivity, u).passed
    assert res.variant is tb.VariantId.B and res.ledger.flops_per_elem == 3108


@pytest.mark.gpu
@pytest.mark.parametrize("variant", VARIANTS)
def test_zero_velocity_is_exactly_zero(variant):
    m = tb.generate_box_mesh(2, 2, 2)
    res = tb.ASSEMBLERS[variant](m, np.zeros((m.n_nodes, 3)), P, tb.RunConfig())
    np.testing.assert_array_equal(res.rhs, np.zeros_like(res.rhs))
    assert res.ledger.flops_per_elem > 0 and res.wall_time > 0.0
    assert res.elements_per_second == pytest.approx(m.n_elems / res.wall_time, rel=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", VARIANTS)
def test_fixed_config_reruns_bitwise_identical(variant):
    m = tb.generate_box_mesh(3, 2, 2)
    u = tb.make_velocity(m, "taylor-green")
    cfg = tb.RunConfig(vector_dim=8, n_threads=2)
    first = tb.ASSEMBLERS[variant](m, u, P, cfg).rhs
    second = tb.ASSEMBLERS[variant](m, u, P, cfg).rhs
    np.testing.assert_array_equal(first, second)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", VARIANTS)
def test_chunk_and_thread_invariance(variant):
    m = tb.generate_box_mesh(3, 2, 2)
    u = tb.make_velocity(m, "taylor-green")
    base = tb.ASSEMBLERS[variant](m, u, P, tb.RunConfig(vector_dim=16)).rhs
    scale = max(np.abs(base).max(), 1e-300)
    for cfg in (tb.RunConfig(vector_dim=1), tb.RunConfig(vector_dim=4096), tb.RunConfig(n_threads=4),
                tb.RunConfig(scatter="atomic"), tb.RunConfig(scatter="colored")):
        rhs = tb.ASSEMBLERS[variant](m, u, P, cfg).rhs
        assert np.abs(rhs - base).max() <= 1e-12 * scale


@pytest.mark.gpu
def test_remainder_and_precolored(oracle):
    m = tb.generate_box_mesh(3, 3, 3)  # 162 elements: a remainder chunk at vector_dim 16
    u = tb.make_velocity(m, "random:4")
    ref = oracle.assemble_reference(m.coords, m.connectivity, u)
    assert tb.verify_variants(m, u, P, tb.RunConfig(vector_dim=16), oracle=ref).passed
    mc = tb.color_elements(tb.generate_box_mesh(2, 2, 2))
    u = tb.make_velocity(mc, "random:2")
    ref = oracle.assemble_reference(mc.coords, mc.connectivity, u)
    for variant in VARIANTS:
        rhs = tb.ASSEMBLERS[variant](mc, u, P, tb.RunConfig(scatter="colored")).rhs
        assert tb.oracle_compare(mc, u, P, rhs, variant, oracle=ref).passed


@pytest.mark.gpu
def test_verify_report_shape_and_default_cross_check():
    """Without an external oracle vector the B shape is the cross-check."""
    m = tb.generate_box_mesh(2, 2, 2)
    u = tb.make_velocity(m, "random:1")
    report = tb.verify_variants(m, u, P)
    assert report.passed and len(report.checks) == 3
    assert {c.variant for c in report.checks} == set(tb.VariantId)
    for c in report.checks:
        assert c.rel_diff <= tb.REL_TOL


@pytest.mark.gpu
def test_fault_injection_detected(golden_small):
    m = tb.generate_box_mesh(2, 2, 2)
    u = golden_small["u_2x2x2_random"]
    report = tb.verify_variants(m, u, P, fault_inject="rs", oracle=golden_small["oracle_2x2x2_random"])
    assert not report.passed
    failed = {c.variant.value: c for c in report.checks if not c.passed}
    assert set(failed) == {"rs"}
    assert failed["rs"].max_abs_diff > 0.0 and failed["rs"].worst_node == 0


@pytest.mark.gpu
def test_empty_mesh_assembles_to_nothing():
    m = tb.Mesh(coords=np.array([[0.0, 0, 0], [1.0, 0, 0]]), connectivity=np.zeros((0, 4), np.int64))
    for fn in tb.ASSEMBLERS.values():
        np.testing.assert_array_equal(fn(m, np.zeros((2, 3)), P, tb.RunConfig()).rhs, np.zeros((2, 3)))


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["b", "rs"])
def test_shapes_mid_size_and_permuted(oracle, golden_mid, golden_small, shape):
    fn = tb.ASSEMBLERS[tb.VariantId(shape)]
    m = tb.generate_box_mesh(16, 16, 16)
    u = tb.make_velocity(m, "random:1")
    for scatter in ("private", "atomic"):
        rhs = fn(m, u, P, tb.RunConfig(scatter=scatter)).rhs
        assert oracle.compare(rhs, golden_mid["rsp_16_random"], m.coords, m.connectivity, u).passed
    pm = tb.Mesh(coords=golden_small["perm6_coords"], connectivity=golden_small["perm6_conn"])
    u = golden_small["perm6_u"]
    rhs = fn(pm, u, P, tb.RunConfig(renumber="none", element_order="keep")).rhs
    assert oracle.compare(rhs, golden_small["perm6_oracle"], pm.coords, pm.connectivity, u).passed


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["b", "rs"])
def test_shapes_device_resident_run(oracle, shape):
    m = tb.generate_box_mesh(6, 5, 4)
    u = tb.make_velocity(m, "random:7")
    asm = tb.Assembler(m, tb.RunConfig(scatter="atomic"))
    asm.set_velocity_host(u)
    assert asm.run(P, variant=tb.VariantId(shape)) >= 1
    rhs = asm.get_rhs_host()
    asm.synchronize()
    ref = oracle.assemble_reference(m.coords, m.connectivity, u)
    assert oracle.compare(rhs, ref, m.coords, m.connectivity, u).passed
    with pytest.raises(RuntimeError):  # colour-by-colour needs a colouring
        asm.run(P, scatter="colored", variant=tb.VariantId(shape))
    asm.close()


# ---------------------------------------------------------------------------
# CPU: the B200 roofline figures (perfmodel)
# ---------------------------------------------------------------------------

def test_perfmodel_b200_ceilings_and_bounds():
    from paper_2403_08777_b200 import perfmodel as pm
    assert pm.B200.balance == pytest.approx(33.48 / 6.5542)
    k = {r["kernel"]: r for r in pm.report()}
    # the production kernel is FP64-compute bound, the baseline shape memory bound
    assert k["RSP-star"]["bound"] == "fp64" and k["B"]["bound"] == "hbm"
    assert 0.3 < k["RSP-star"]["frac"] < 1.0
    assert k["RSP-star"]["measured_gelem_s"] > 3 * k["RSP"]["measured_gelem_s"]
    # ceiling = min(compute, memory) per element
    star = pm.SHAPES_128[-1]
    assert pm.attainable_elem_per_s(star) == pytest.approx(
        min(33.48e12 / star.flop, 6.5542e12 / star.dram_bytes))
    with pytest.raises(ValueError):
        pm.attainable_elem_per_s(pm.Kernel("x", 1.0, 0.0))


@pytest.mark.gpu
@pytest.mark.parametrize("scatter", ["atomic", "colored"])
def test_study_shape_p_matches_oracle(oracle, scatter):
    """The study-only "P" shape (B statements, literal trip counts)."""
    m = tb.generate_box_mesh(7, 6, 5)
    u = tb.make_velocity(m, "random:3")
    asm = tb.Assembler(m, tb.RunConfig(scatter=scatter), build_colors=True)
    rhs, _ = asm.assemble(u, P, variant="p")
    ref = oracle.assemble_reference(m.coords, m.connectivity, u)
    assert oracle.compare(rhs, ref, m.coords, m.connectivity, u).passed
    with pytest.raises(ValueError):
        asm.assemble(u, P, variant="q")
    asm.close()

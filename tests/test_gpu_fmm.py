"""Laplace FMM on the GPU vs the reference SummationPlan (oracle/_ref), the
restatement and long-double direct sums (summation.cpp:224-348, 610-643)."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_2203_05933_b200 import workloads as W

pytestmark = pytest.mark.gpu


def lap(vp):
    return vp.make_kernel(vp.KernelFamily.Laplace)


def test_cfg1_fmm_vs_reference(vp, ref, rest):
    w = W.cfg1()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        assert plan.levels() == 5 and plan.expansion_order() == 50
        gpu = plan.apply(w.q)
        again = plan.apply(w.q)
    assert np.array_equal(gpu, again)  # run-to-run bit identical
    rp = ref.plan(0, 0.0, w.src, w.tgt, 1e-12)
    cpu = rp.apply(w.q)
    assert rel_l2(gpu, cpu) <= 1e-13
    ld = rest.pairwise_ld(0, 0.0, w.src, w.q, w.tgt)
    assert rel_l2(gpu, ld) <= 1e-12


def test_cfg2_fmm_vs_reference(vp, rest):
    w = W.cfg2()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        assert plan.levels() == 7
        gpu = plan.apply(w.q)
    cpu = rest.plan_sum(0, 0.0, w.src, w.q, w.tgt, 1e-12)
    assert rel_l2(gpu, cpu) <= 1e-13
    idx = np.random.default_rng(0).choice(w.nt, 2000, replace=False)
    ld = rest.pairwise_ld(0, 0.0, w.src, w.q, w.tgt[idx])
    assert rel_l2(gpu[idx], ld) <= 1e-12


@pytest.mark.parametrize("eps", [1e-3, 1e-4, 1e-6, 1e-7, 1e-9, 1e-11])
def test_tolerances(vp, rest, eps):
    """Every order between the clamps (P = 16 at 1e-3 ... 50 at 1e-12): the P2M
    quarters (ceil(P/4) = 4 ... 13 powers per lane), the M2L instances with a
    compile-time k-step count (P = 27, 39, 50) and the generic ones."""
    w = W.cfg1()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, eps) as plan:
        gpu = plan.apply(w.q)
    cpu = rest.plan_sum(0, 0.0, w.src, w.q, w.tgt, eps)
    ld = rest.pairwise_ld(0, 0.0, w.src, w.q, w.tgt)
    assert rel_l2(gpu, cpu) <= 1e-13
    assert rel_l2(gpu, ld) <= eps


def test_spec_acceptance8_random_1e4(vp, rest):
    """1e4 random points, eps=1e-10 -> rel l2 <= 1e-10 vs direct."""
    rng = np.random.default_rng(8)
    pts = rng.uniform(0, 1, (10_000, 2))
    q = rng.standard_normal(10_000)
    gpu = None
    with vp.SummationPlan(lap(vp), pts, pts, 1e-10) as plan:
        assert plan.levels() > 0
        gpu = plan.apply(q)
    ld = rest.pairwise_ld(0, 0.0, pts, q, pts)
    assert rel_l2(gpu, ld) <= 1e-10


def test_zero_charges_and_linearity(vp):
    rng = np.random.default_rng(9)
    pts = rng.uniform(-1, 1, (20_000, 2))
    tg = rng.uniform(-1, 1, (15_000, 2))
    with vp.SummationPlan(lap(vp), pts, tg, 1e-12) as plan:
        assert np.all(plan.apply(np.zeros(20_000)) == 0.0)
        q1 = rng.choice([-1.0, 1.0], 20_000)  # Rademacher
        q2 = rng.standard_normal(20_000)
        a, b, ab = plan.apply(q1), plan.apply(q2), plan.apply(q1 + q2)
    assert rel_l2(ab, a + b) <= 10 * 1e-12


def test_single_source(vp, rest):
    rng = np.random.default_rng(10)
    tg = rng.uniform(-1, 1, (5000, 2))
    src = np.concatenate([[[0.3, -0.2]], rng.uniform(-1, 1, (999, 2))])
    q = np.zeros(1000)
    q[0] = 1.0
    with vp.SummationPlan(lap(vp), src, tg, 1e-12) as plan:
        gpu = plan.apply(q)
    d = tg - src[0]
    exact = -0.25 / np.pi * np.log(d[:, 0] ** 2 + d[:, 1] ** 2)
    assert rel_l2(gpu, exact) <= 1e-13


def test_apply_size_mismatch_message(vp):
    pts = np.random.default_rng(1).uniform(0, 1, (3000, 2))
    with vp.SummationPlan(lap(vp), pts, pts, 1e-12) as plan:
        with pytest.raises(vp.InvalidArgument,
                           match="SummationPlan::apply: charge count 5 does not match source count 3000"):
            plan.apply(np.ones(5))


def test_pairwise_mode(vp, rest):
    rng = np.random.default_rng(12)
    src = rng.uniform(0, 1, (1500, 2))
    tgt = np.concatenate([src[:500], rng.uniform(0, 1, (1000, 2))])  # coincident -> skipped
    q = rng.standard_normal(1500)
    with vp.SummationPlan(lap(vp), src, tgt, 1e-12) as plan:
        assert plan.levels() == 0 and plan.expansion_order() == 0
        gpu = plan.apply(q)
    cpu = rest.plan_sum(0, 0.0, src, q, tgt, 1e-12)
    assert rel_l2(gpu, cpu) <= 1e-14


def test_native_mode_deeper_tree(vp, rest):
    w = W.cfg3()
    sub = slice(0, None, 4)
    src, q = w.src[sub], w.q[sub]
    with vp.SummationPlan(lap(vp), src, src, 1e-12, mode="native") as plan:
        gpu = plan.apply(q)
    idx = np.random.default_rng(5).choice(len(src), 1500, replace=False)
    ld = rest.pairwise_ld(0, 0.0, src, q, src[idx])
    assert rel_l2(gpu[idx], ld) <= 1e-12


def test_device_pointer_apply(vp):
    torch = pytest.importorskip("torch")
    w = W.cfg1()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        host = plan.apply(w.q)
        qd = torch.tensor(w.q, device="cuda")
        od = torch.empty(w.nt, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream()
        plan.apply_device(qd.data_ptr(), od.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(od.cpu().numpy(), host)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_target_shards_assemble_bit_exact(vp, world):
    """Multi-GPU sharding emulated shard by shard on one GPU: the sum of the
    shards' outputs equals the single-plan result bit for bit."""
    from paper_2203_05933_b200 import multigpu
    w = W.cfg2()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        full = plan.apply(w.q)
        total = np.zeros_like(full)
        seen = np.zeros(w.nt, bool)
        t = plan.dump_tree()
        for r in range(world):
            lo, hi = multigpu.shard_plan(plan, r, world)
            part = plan.apply(w.q)
            own = multigpu.owned_targets(t["tgt_off"], t["tgt_ids"], (lo, hi))
            mask = np.ones(w.nt, bool)
            mask[own] = False
            assert np.all(part[mask] == 0.0)
            assert not seen[own].any()
            seen[own] = True
            total += part
        plan.set_shard(0, 4 ** plan.levels())
        assert seen.all()
        assert np.array_equal(total, full)
        assert np.array_equal(plan.apply(w.q), full)


@pytest.mark.parametrize("env", [("VPG_MULTILEVEL", "0"), ("VPG_MULTILEVEL", "1"),
                                 ("VPG_PASS_CAP", "64"), ("VPG_PASS_CAP", "1024")])
def test_chain_multilevel_and_hybrid_passes(vp, rest, monkeypatch, env):
    """Upward/downward passes as level chains (M2M/L2L, the reference
    structure), as direct per-level P2M/L2P (multilevel), or hybrid (direct
    below a box-size threshold, shifts above) agree with the oracle to the
    same tolerance."""
    monkeypatch.setenv(*env)
    w = W.cfg2()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        gpu = plan.apply(w.q)
    cpu = rest.plan_sum(0, 0.0, w.src, w.q, w.tgt, 1e-12)
    assert rel_l2(gpu, cpu) <= 1e-13


def test_graph_cache_pointer_pairs_and_profiling_agree(vp):
    """Device-pointer applies are replayed from a per-(q, out) CUDA graph;
    more pointer pairs than cache slots, host-pointer applies and the
    profiled (plain-launch) path all give bit-identical potentials."""
    torch = pytest.importorskip("torch")
    w = W.cfg2()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        ref = plan.apply(w.q)
        s = torch.cuda.current_stream()
        qd = torch.tensor(w.q, device="cuda")
        outs = [torch.empty(w.nt, dtype=torch.float64, device="cuda") for _ in range(11)]
        for rep in range(2):
            for o in outs:
                o.fill_(float("nan"))
                plan.apply_device(qd.data_ptr(), o.data_ptr(), s.cuda_stream)
            torch.cuda.synchronize()
            for o in outs:
                assert np.array_equal(o.cpu().numpy(), ref)
        plan.set_profiling(True)
        prof = plan.apply(w.q)
        plan.set_profiling(False)
        assert np.array_equal(prof, ref)


def test_concurrent_host_threads(vp):
    """apply is const and may run from several host threads at once
    (summation.hpp:32-33): every thread gets the single-thread result."""
    import threading
    w = W.cfg1()
    rng = np.random.default_rng(3)
    qs = [rng.standard_normal(w.ns) for _ in range(6)]
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        want = [plan.apply(q) for q in qs]
        got = [None] * len(qs)

        def run(i):
            for _ in range(3):
                got[i] = plan.apply(qs[i])

        th = [threading.Thread(target=run, args=(i,)) for i in range(len(qs))]
        for t in th:
            t.start()
        for t in th:
            t.join()
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_rademacher_charges(vp, rest):
    """SPEC.md:520-523 invariants: Rademacher (+-1) charges on random points
    against the long-double direct sum."""
    rng = np.random.default_rng(77)
    pts = rng.uniform(-1, 1, (40_000, 2))
    q = rng.choice([-1.0, 1.0], size=40_000)
    with vp.SummationPlan(lap(vp), pts, pts, 1e-10) as plan:
        gpu = plan.apply(q)
    idx = rng.choice(40_000, 1000, replace=False)
    ld = rest.pairwise_ld(0, 0.0, pts, q, pts[idx])
    assert rel_l2(gpu[idx], ld) <= 1e-10


def test_runtime_ratio_50k_to_100k(vp):
    """doubling N from 50k to 100k costs at most 2.6x (device
    time of the apply, median of 5)."""
    import time
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(78)
    t = {}
    for n in (50_000, 100_000):
        pts = rng.uniform(-1, 1, (n, 2))
        q = rng.standard_normal(n)
        with vp.SummationPlan(lap(vp), pts, pts, 1e-10) as plan:
            qd = torch.tensor(q, device="cuda")
            od = torch.empty(n, dtype=torch.float64, device="cuda")
            s = torch.cuda.current_stream()
            for _ in range(3):
                plan.apply_device(qd.data_ptr(), od.data_ptr(), s.cuda_stream)
            ms = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.apply_device(qd.data_ptr(), od.data_ptr(), s.cuda_stream)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            t[n] = sorted(ms)[2]
    assert t[100_000] / t[50_000] <= 2.6, t


@pytest.mark.parametrize("mode", ["reference", "native"])
def test_near_field_zero_and_subnormal_pairs(vp, rest, mode):
    """The near-field hot loop has no zero test; the plan lists the pairs with
    r^2 zero (skipped, summation.cpp:340) or subnormal (exact log) and the
    apply corrects them.  Points next to the origin make subnormal r^2."""
    rng = np.random.default_rng(41)
    src = np.concatenate([rng.uniform(-1, 1, (20_000, 2)), [[0.0, 0.0], [0.0, 3e-160]]])
    tgt = np.concatenate([src[:400], [[1e-160, 0.0], [0.0, 0.0], [-2e-161, 1e-161]],
                          rng.uniform(-1, 1, (3000, 2))])
    q = rng.standard_normal(len(src))
    with vp.SummationPlan(lap(vp), src, tgt, 1e-12, mode=mode) as plan:
        gpu = plan.apply(q)
    cpu = rest.plan_sum(0, 0.0, src, q, tgt, 1e-12)
    assert rel_l2(gpu, cpu) <= 1e-12
    # the three targets at the origin carry log(r^2) ~ -737 terms
    assert np.allclose(gpu[400:403], cpu[400:403], rtol=1e-12, atol=0)


@pytest.mark.parametrize("sym,smin", [("0", None), ("1", "0"), ("1", "64")])
def test_symmetric_near_field(vp, rest, monkeypatch, sym, smin):
    """'Targets = nodes' plans may evaluate each unordered near pair once
    (plan.cuh SymTask), for every pair (VPG_SYM_MIN=0) or only for pairs of
    leaves with >= 64 sources (hybrid).  Off, full and hybrid, cfg2 (nodes +
    10,000 unmatched targets) matches the oracle, and shards still assemble
    bit-exactly."""
    from paper_2203_05933_b200 import multigpu
    monkeypatch.setenv("VPG_SYM", sym)
    if smin is not None:
        monkeypatch.setenv("VPG_SYM_MIN", smin)
    w = W.cfg2()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        assert plan.info()["near_symmetric"] == (1 if sym == "1" else 0)
        gpu = plan.apply(w.q)
        total = np.zeros_like(gpu)
        for r in range(3):
            multigpu.shard_plan(plan, r, 3)
            total += plan.apply(w.q)
        plan.set_shard(0, 4 ** plan.levels())
        assert np.array_equal(total, gpu)
        assert np.array_equal(plan.apply(w.q), gpu)
    cpu = rest.plan_sum(0, 0.0, w.src, w.q, w.tgt, 1e-12)
    assert rel_l2(gpu, cpu) <= 1e-13


@pytest.mark.parametrize("sym,extra", [("0", True), ("1", True), ("1", False)])
def test_symmetric_near_field_duplicates_and_subnormal(vp, rest, monkeypatch, sym, extra):
    """Coincident distinct sources and subnormal r^2 with targets = sources
    (+ extras): the symmetric path feeds each pair to both targets and the
    coincidence list undoes exactly what the hot loop added.  Without extras
    the finalize runs without the smem table (global-table fix-ups)."""
    monkeypatch.setenv("VPG_SYM", sym)
    rng = np.random.default_rng(43)
    base = rng.uniform(-1, 1, (30_000, 2))
    src = np.concatenate([base, base[:500], [[0.0, 0.0], [0.0, 3e-160], [1e-160, 0.0]]])
    tgt = np.concatenate([src, rng.uniform(-1, 1, (2000, 2)), [[-2e-161, 1e-161]]]) if extra else src.copy()
    q = rng.standard_normal(len(src))
    with vp.SummationPlan(lap(vp), src, tgt, 1e-12) as plan:
        gpu = plan.apply(q)
    cpu = rest.plan_sum(0, 0.0, src, q, tgt, 1e-12)
    assert rel_l2(gpu, cpu) <= 1e-12
    n = len(src)
    assert np.allclose(gpu[n - 3:n], cpu[n - 3:n], rtol=1e-12, atol=0)


@pytest.mark.parametrize("sym", ["0", "1"])
def test_subnormal_pairs_across_leaf_edges(vp, rest, monkeypatch, sym):
    """Points in a 1e-152 square: nearest neighbours are ~1e-155 apart, so
    many near pairs have subnormal r^2, and with leaves ~3e-154 wide many of
    them straddle a leaf edge.  The plan's coincidence scan covers every near
    range (not just the own leaf), so each such pair gets the reference's
    exact log (summation.cpp:340-341) in both near-field paths."""
    monkeypatch.setenv("VPG_SYM", sym)
    rng = np.random.default_rng(44)
    pts = rng.uniform(0.0, 1e-152, (20_000, 2))
    q = rng.standard_normal(len(pts))
    with vp.SummationPlan(lap(vp), pts, pts, 1e-12) as plan:
        assert plan.levels() > 0
        gpu = plan.apply(q)
    cpu = rest.plan_sum(0, 0.0, pts, q, pts, 1e-12)
    assert rel_l2(gpu, cpu) <= 1e-13


def _lattice_points(nbox, nx, ny):
    """nbox x nbox boxes on [-1, 1]^2, each an nx x ny tensor Gauss-Legendre rule."""
    h = 2.0 / nbox
    gx, _ = np.polynomial.legendre.leggauss(nx)
    gy, _ = np.polynomial.legendre.leggauss(ny)
    c = -1.0 + (np.arange(nbox) + 0.5) * h
    X = (c[None, :, None, None] + 0.5 * h * gx[None, None, None, :]) + 0.0 * c[:, None, None, None] + 0.0 * gy[None, None, :, None]
    Y = (c[:, None, None, None] + 0.5 * h * gy[None, None, :, None]) + 0.0 * c[None, :, None, None] + 0.0 * gx[None, None, None, :]
    return np.stack([X.ravel(), Y.ravel()], axis=1)


@pytest.mark.parametrize("nx,ny,m", [(8, 8, 64), (16, 8, 128)])
def test_lattice_near_field(vp, rest, monkeypatch, nx, ny, m):
    """Leaves that are translates of one point pattern (one box per leaf, 64 or
    128 nodes): the near field runs as dense K_o q products (lattice.cu) and
    agrees with the pairwise kernels to rounding and with the oracle; shards
    assemble bit-exactly; one node moved by 1e-9 sends the plan back to the
    pairwise kernels."""
    from paper_2203_05933_b200 import multigpu
    pts = _lattice_points(128, nx, ny)
    rng = np.random.default_rng(77)
    q = rng.standard_normal(len(pts)) * np.exp(-3.0 * (pts[:, 0] ** 2 + pts[:, 1] ** 2))
    with vp.SummationPlan(lap(vp), pts, pts, 1e-12) as plan:
        info = plan.info()
        assert info["levels"] == 7 and info["near_lattice"] == 1
        lat = plan.apply(q)
        total = np.zeros_like(lat)
        for r in range(3):
            multigpu.shard_plan(plan, r, 3)
            total += plan.apply(q)
        plan.set_shard(0, 4 ** plan.levels())
        assert np.array_equal(total, lat)
        assert np.array_equal(plan.apply(q), lat)
    monkeypatch.setenv("VPG_LATTICE_P2M", "0")  # the lattice near field with the pairwise P2M kernel
    with vp.SummationPlan(lap(vp), pts, pts, 1e-12) as plan:
        assert plan.info()["near_lattice"] == 1
        lat_p2m0 = plan.apply(q)
    monkeypatch.delenv("VPG_LATTICE_P2M")
    assert rel_l2(lat, lat_p2m0) <= 1e-14
    monkeypatch.setenv("VPG_LATTICE", "0")
    with vp.SummationPlan(lap(vp), pts, pts, 1e-12) as plan:
        assert plan.info()["near_lattice"] == 0
        pair = plan.apply(q)
    assert rel_l2(lat, pair) <= 1e-14
    monkeypatch.delenv("VPG_LATTICE")
    if m == 64:
        cpu = rest.plan_sum(0, 0.0, pts, q, pts, 1e-12)
        assert rel_l2(lat, cpu) <= 1e-13
    moved = pts.copy()
    moved[12345, 0] += 1e-9
    with vp.SummationPlan(lap(vp), moved, moved, 1e-12) as plan:
        assert plan.info()["near_lattice"] == 0
        gpu = plan.apply(q)
    assert rel_l2(gpu, pair) <= 1e-9 and not np.array_equal(gpu, pair)


@pytest.mark.parametrize("eps", [1e-12, 1e-6, 1e-4])
def test_m2l_by_offset_agrees(vp, monkeypatch, eps):
    """The opt-in M2L batched by offset (m2lgrid.cu, VPG_M2L_GRID=1): same
    factorisation, same arithmetic per list entry and same order of the entry
    sums as the per-target-box kernel, so the potentials agree to rounding -- on
    cfg2 (irregular occupancy, empty boxes, domain edges) and on a shard."""
    from paper_2203_05933_b200 import multigpu
    w = W.cfg2()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, eps) as plan:
        box = plan.apply(w.q)
        multigpu.shard_plan(plan, 1, 3)
        box_shard = plan.apply(w.q)
    monkeypatch.setenv("VPG_M2L_GRID", "1")
    with vp.SummationPlan(lap(vp), w.src, w.tgt, eps) as plan:
        grid = plan.apply(w.q)
        multigpu.shard_plan(plan, 1, 3)
        grid_shard = plan.apply(w.q)
    assert rel_l2(grid, box) <= 1e-14
    assert rel_l2(grid_shard, box_shard) <= 1e-14
    assert np.array_equal(grid_shard != 0.0, box_shard != 0.0)

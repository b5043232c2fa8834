"""the general Array-OL repetitive task (arbitrary tilers, S:65-70,
S:248-252, executed as S:517-520) and SPEC's launch topology rule
(S:349-357).  Topology tests are host-only; task/coverage parity runs on the
GPU against the oracle's general task executor."""
import numpy as np
import pytest

import oracle
import paper_1103_4881_b200 as ds
import synth
from conftest import FUZZ_SCALE, fuzz_seed


# ---------------------------------------------------------------- topology --
def test_topology_spec_examples():
    # S:355 multiplicity [288,44], max_wg 256 -> local [16,16], global [288,48], guarded
    t = ds.ds_compute_topology([288, 44], max_wg=256)
    assert t == dict(multiplicity=[288, 44], local=[16, 16], global_=[288, 48], guarded=True)
    # S:356 multiplicity [8], min_items 64 -> local [8], global [8], not guarded
    t = ds.ds_compute_topology([8], max_wg=256)
    assert t == dict(multiplicity=[8], local=[8], global_=[8], guarded=False)
    # S:357 [2,3,4,5] on a 3-dim device -> collapsed to [2,3,20]
    assert ds.ds_compute_topology([2, 3, 4, 5], max_dims=3)["multiplicity"] == [2, 3, 20]


def test_topology_invariants_random():
    """product(local) <= max_wg, global multiple of local, product(global)
    >= product(multiplicity), padding < 2x when product >= min_items."""
    rng = np.random.default_rng(651)
    for _ in range(1000):
        nd = int(rng.integers(1, 5))
        mult = [int(rng.integers(1, 400)) for _ in range(nd)]
        max_wg = int(rng.choice([32, 64, 100, 256, 1024]))
        max_dims = int(rng.integers(1, 4))
        t = ds.ds_compute_topology(mult, max_wg=max_wg, max_dims=max_dims)
        m, loc, glob = t["multiplicity"], t["local"], t["global_"]
        assert len(m) == min(nd, max_dims)
        assert int(np.prod(m)) == int(np.prod(mult))
        assert int(np.prod(loc)) <= max_wg
        assert all(g % l == 0 and g >= mm for g, l, mm in zip(glob, loc, m))
        assert t["guarded"] == (glob != m)
        if int(np.prod(m)) >= 64:
            assert int(np.prod(glob)) < 2 * int(np.prod(m))


def test_topology_errors():
    with pytest.raises(ds.DSError):
        ds.ds_compute_topology([4, 4], max_wg=0)          # S:354 zero max work-group -> error
    with pytest.raises(ds.DSError):
        ds.ds_compute_topology([0])


# ------------------------------------------------------------ GPU parity --
torch = pytest.importorskip("torch")


def _exact_out_tiler(rng, nrep_shape, npat_shape):
    """An exact-cover output tiler of a 2-D array for the given repetition and
    pattern shapes (1-D each): blocked, transposed or interleaved, random origin."""
    r, p = nrep_shape[0], npat_shape[0]
    kind = int(rng.integers(0, 3))
    if kind == 0:      # rows of blocks: out[r][f]
        shape, pav, fit = (r, p), [[1], [0]], [[0], [1]]
    elif kind == 1:    # transposed: out[f][r]
        shape, pav, fit = (p, r), [[0], [1]], [[1], [0]]
    else:              # interleaved 1-D: out[r + R f]
        shape, pav, fit = (r * p,), [[1]], [[r]]
    origin = [int(rng.integers(-50, 50)) for _ in shape]
    return shape, oracle.make_tiler(shape, origin, pav, fit, [p]), ds.make_tiler(shape, origin, pav, fit, [p])


@pytest.mark.gpu
@pytest.mark.parametrize("policy", [ds.DS_TOPO_FLAT, ds.DS_TOPO_SPEC])
def test_run_task_random_tilers(policy):
    rng = np.random.default_rng(fuzz_seed(77 + policy))
    for trial in range(60 * FUZZ_SCALE):
        nd = int(rng.integers(1, 4))
        in_shape = [int(rng.integers(1, 30)) for _ in range(nd)]
        R = int(rng.integers(1, 200))
        P = int(rng.integers(1, 17))
        Q = int(rng.integers(1, 9))
        origin = [int(rng.integers(-100, 100)) for _ in range(nd)]
        pav = [[int(rng.integers(-7, 8))] for _ in range(nd)]
        fit = [[int(rng.integers(-5, 6))] for _ in range(nd)]
        tin_o = oracle.make_tiler(in_shape, origin, pav, fit, [P])
        tin_d = ds.make_tiler(in_shape, origin, pav, fit, [P])
        out_shape, tout_o, tout_d = _exact_out_tiler(rng, [R], [Q])
        w = [[int(x) for x in rng.integers(-20, 60, P)] for _ in range(Q)]
        D, B = int(rng.integers(1, 50)), int(rng.integers(-100, 100))
        body_o = oracle.make_stage(P, P, 0, w, D, B)
        body_d = ds.make_body(w, D, B, n_in=P)
        a = rng.integers(0, 256, in_shape).astype(np.uint8)
        want = oracle.run_task(a, tin_o, out_shape, tout_o, [R], body_o)
        x = torch.from_numpy(a).cuda()
        y = torch.zeros(out_shape, dtype=torch.uint8, device="cuda")
        ds.run_task(x, tin_d, y, tout_d, [R], body_d, policy=policy)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), want), (trial, in_shape, R, P, Q)


@pytest.mark.gpu
@pytest.mark.parametrize("policy", [ds.DS_TOPO_FLAT, ds.DS_TOPO_SPEC])
def test_run_task_downscaler_tasks(policy):
    """The paper's yhfk task (multiplicity [288,44]) and its V task
    through the general executor equal the dedicated kernels and the oracle."""
    W, H = 352, 288
    plane = synth.random_frames(3, 0, 1, W, H, 1)[0].reshape(H, W)
    mid_o, out_o = oracle.execute_plane_mid(plane)
    spec = ds.ds_default_spec()
    hw = [[spec.h.weight[k][i] for i in range(8)] for k in range(3)]
    vw = [[spec.v.weight[k][i] for i in range(9)] for k in range(4)]
    x = torch.from_numpy(plane).cuda()
    mid = torch.zeros((H, 132), dtype=torch.uint8, device="cuda")
    out = torch.zeros((128, 132), dtype=torch.uint8, device="cuda")
    ds.run_task(x, ds.make_tiler((H, W), (0, 0), [[1, 0], [0, 8]], [[0], [1]], [8]), mid,
                ds.make_tiler((H, 132), (0, 0), [[1, 0], [0, 3]], [[0], [1]], [3]), [288, 44],
                ds.make_body(hw, 6, 3, n_in=8), policy=policy)
    ds.run_task(mid, ds.make_tiler((H, 132), (0, 0), [[9, 0], [0, 1]], [[1], [0]], [9]), out,
                ds.make_tiler((128, 132), (0, 0), [[4, 0], [0, 1]], [[1], [0]], [4]), [32, 132],
                ds.make_body(vw, 8, 4, n_in=9), policy=policy)
    torch.cuda.synchronize()
    assert np.array_equal(mid.cpu().numpy(), mid_o)
    assert np.array_equal(out.cpu().numpy(), out_o)


@pytest.mark.gpu
def test_tiler_coverage_matches_oracle():
    # S:284-286 examples plus random tilers; classification and counts
    cases = [((288, 132), (0, 0), [[1, 0], [0, 3]], [[0], [1]], [3], (288, 44), "exact"),
             ((352,), (0,), [[4]], [[1]], [8], (88,), "overlaps"),
             ((12,), (0,), [[4]], [[1]], [3], (3,), "gaps")]
    for shape, origin, pav, fit, pat, rep, kind in cases:
        got = ds.tiler_coverage(ds.make_tiler(shape, origin, pav, fit, pat), rep)
        assert got[0] == kind
        assert oracle.check_coverage(oracle.make_tiler(shape, origin, pav, fit, pat), rep)[0] == kind
    assert ds.tiler_coverage(ds.make_tiler((12,), (0,), [[4]], [[1]], [3]), (3,))[2] == 3
    rng = np.random.default_rng(9)
    for _ in range(100):
        nd = int(rng.integers(1, 3))
        shape = [int(rng.integers(1, 20)) for _ in range(nd)]
        rep = [int(rng.integers(1, 6))]
        pat = [int(rng.integers(1, 5))]
        origin = [int(rng.integers(-9, 9)) for _ in range(nd)]
        pav = [[int(rng.integers(-4, 5))] for _ in range(nd)]
        fit = [[int(rng.integers(-3, 4))] for _ in range(nd)]
        counts = np.zeros(shape, np.int64)
        for r in range(rep[0]):
            for f in range(pat[0]):
                idx = tuple((o + p[0] * r + q[0] * f) % s for o, p, q, s in zip(origin, pav, fit, shape))
                counts[idx] += 1
        kind, over, gaps = ds.tiler_coverage(ds.make_tiler(shape, origin, pav, fit, pat), rep)
        assert over == int((counts > 1).sum()) and gaps == int((counts == 0).sum())
        assert kind == oracle.check_coverage(oracle.make_tiler(shape, origin, pav, fit, pat), rep)[0]


@pytest.mark.gpu
def test_run_task_errors():
    x = torch.zeros(16, dtype=torch.uint8, device="cuda")
    y = torch.zeros(16, dtype=torch.uint8, device="cuda")
    t = ds.make_tiler((16,), (0,), [[1]], [[0]], [])
    with pytest.raises(ds.DSError):          # body arity mismatch
        ds.run_task(x, t, y, t, [16], ds.make_body([[1, 1]], n_in=2))
    with pytest.raises(ds.DSError):          # in and out overlap
        ds.run_task(x, t, x, t, [16], ds.make_body([[1]], n_in=1))


@pytest.mark.gpu
@pytest.mark.parametrize("policy", [ds.DS_TOPO_FLAT, ds.DS_TOPO_SPEC])
def test_run_task_large_extents(policy):
    """Large, odd extents exercise the 32-bit multiply-high divisions (and a
    3-D repetition space with frames as its outer dimension)."""
    rng = np.random.default_rng(12)
    n, H, W = 3, 999, 1000003 // 1000 * 8      # W = 8000
    a = rng.integers(0, 256, (n, H, W)).astype(np.uint8)
    tin_args = ((n, H, W), (1, -3, 5), [[1, 0, 0], [0, 1, 0], [0, 0, 8]], [[0], [0], [1]], [8])
    tout_args = ((n, H, W // 8 * 3), (0, 7, 0), [[1, 0, 0], [0, 1, 0], [0, 0, 3]], [[0], [0], [1]], [3])
    w = [[1, 5, 0, 0, 0, 0, 0, 0], [0, 0, 0, 3, 3, 0, 0, 0], [0, 0, 0, 0, 0, 0, 5, 1]]
    want = oracle.run_task(a, oracle.make_tiler(*tin_args), tout_args[0], oracle.make_tiler(*tout_args),
                           [n, H, W // 8], oracle.make_stage(8, 8, 0, w, 6, 3))
    x = torch.from_numpy(a).cuda()
    y = torch.zeros(tout_args[0], dtype=torch.uint8, device="cuda")
    ds.run_task(x, ds.make_tiler(*tin_args), y, ds.make_tiler(*tout_args), [n, H, W // 8],
                ds.make_body(w, 6, 3, n_in=8), policy=policy)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), want)


@pytest.mark.gpu
@pytest.mark.parametrize("rep", [(4096, 2, 1), (2, 4096, 1), (1, 3, 70000)])
def test_run_task_spec_topology_axis_limits(rep):
    """DS_TOPO_SPEC launches whose power-of-two box is large along the first
    dimension (rep [4096, 2, 1] gives local[0] = 128 > the 64-thread block.z
    limit): the launch picks CUDA axes that fit, the result is the oracle's."""
    n0, n1, n2 = rep
    shape = (n0, n1, n2 * 2)
    rng = np.random.default_rng(5)
    a = rng.integers(0, 256, shape).astype(np.uint8)
    tin_args = (shape, (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, 2]], [[0], [0], [1]], [2])
    tout_args = (rep, (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0], [0], [0]], [1])
    w = [[3, 5]]
    want = oracle.run_task(a, oracle.make_tiler(*tin_args), rep, oracle.make_tiler(*tout_args), list(rep),
                           oracle.make_stage(2, 2, 0, w, 8, 4))
    y = torch.zeros(rep, dtype=torch.uint8, device="cuda")
    ds.run_task(torch.from_numpy(a).cuda(), ds.make_tiler(*tin_args), y, ds.make_tiler(*tout_args), list(rep),
                ds.make_body(w, 8, 4, n_in=2), policy=ds.DS_TOPO_SPEC)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), want)


def _affine_in_tiler(rng, in_shape, R, P):
    """A wrap-free 1-rep / 1-pattern input tiler on `in_shape` (possibly with
    negative paving or fitting and a shifted origin): the affine task path."""
    nd = len(in_shape)
    pav, fit, origin = [], [], []
    for d in range(nd):
        s = in_shape[d]
        p = int(rng.integers(-(s // max(R, 1)), s // max(R, 1) + 1)) if R > 1 else int(rng.integers(-3, 4))
        f = int(rng.integers(-(s // max(P, 1)), s // max(P, 1) + 1)) if P > 1 else int(rng.integers(-3, 4))
        lo = min(0, p * (R - 1)) + min(0, f * (P - 1))
        hi = max(0, p * (R - 1)) + max(0, f * (P - 1))
        if hi - lo >= s:
            p, f, lo, hi = 0, 0, 0, 0
        o = int(rng.integers(-lo, s - hi))
        # add multiples of the extent: same tiler mod shape, still affine
        pav.append([p + s * int(rng.integers(-2, 3))])
        fit.append([f + s * int(rng.integers(-2, 3))])
        origin.append(o + s * int(rng.integers(-2, 3)))
    return origin, pav, fit


@pytest.mark.gpu
@pytest.mark.parametrize("policy", [ds.DS_TOPO_FLAT, ds.DS_TOPO_SPEC])
def test_run_task_affine_random(policy):
    """Wrap-free tilers take the affine path (offsets A + a.r + b[e], no
    modulo); results must equal the oracle's modulo tiler semantics."""
    rng = np.random.default_rng(fuzz_seed(4881 + policy))
    for trial in range(60 * FUZZ_SCALE):
        nd = int(rng.integers(1, 4))
        R = int(rng.integers(1, 300))
        P = int(rng.integers(1, 17))
        Q = int(rng.integers(1, 9))
        in_shape = [int(rng.integers(1, 40)) for _ in range(nd)]
        in_shape[-1] = max(in_shape[-1], int(rng.integers(P, 4 * P + 2)))
        origin, pav, fit = _affine_in_tiler(rng, in_shape, R, P)
        tin_o = oracle.make_tiler(in_shape, origin, pav, fit, [P])
        tin_d = ds.make_tiler(in_shape, origin, pav, fit, [P])
        kind = int(rng.integers(0, 2))
        out_shape = (R, Q) if kind == 0 else (Q, R)
        opav, ofit = ([[1], [0]], [[0], [1]]) if kind == 0 else ([[0], [1]], [[1], [0]])
        tout_o = oracle.make_tiler(out_shape, (0, 0), opav, ofit, [Q])
        tout_d = ds.make_tiler(out_shape, (0, 0), opav, ofit, [Q])
        wide = trial % 3 == 0
        w = [[int(x) for x in rng.integers(-300 if wide else -20, 300 if wide else 60, P)] for _ in range(Q)]
        D = int(rng.choice([1, 2, 3, 6, 7, 8, 255, 1000, 65537, 1 << 20]))
        B = int(rng.integers(-100, 100))
        a = rng.integers(0, 256, in_shape).astype(np.uint8)
        want = oracle.run_task(a, tin_o, out_shape, tout_o, [R], oracle.make_stage(P, P, 0, w, D, B))
        x = torch.from_numpy(a).cuda()
        y = torch.zeros(out_shape, dtype=torch.uint8, device="cuda")
        ds.run_task(x, tin_d, y, tout_d, [R], ds.make_body(w, D, B, n_in=P), policy=policy)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), want), (trial, in_shape, origin, pav, fit, R, P, Q, D)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [4, 8, 12, 16])
def test_run_task_affine_words(P):
    """Contiguous, word-aligned patterns with s8 taps take the dense streaming
    path (both tilers row-major runs; 20 full warps of 128 repetitions plus a
    ragged tail) -- a 3-D repetition space, frames outermost, as in the paper's
    yhfk task.  Origins shifted by 1-3 bytes (and an input pointer 1 byte into
    its allocation) take the word path with aligned loads funnelled by the
    misalignment."""
    rng = np.random.default_rng(P)
    n, H, Wp = 3, 37, 24
    W = P * Wp
    a = rng.integers(0, 256, (n, H, W)).astype(np.uint8)
    Q = {4: 1, 8: 3, 12: 5, 16: 8}[P]       # dense path: 128 Q output bytes per warp
    w = [[int(x) for x in rng.integers(-128, 128, P)] for _ in range(Q)]
    for origin, poff in (((0, 0, 0), 0), ((0, 0, 1), 0), ((0, 0, 2), 0), ((0, 0, 3), 0), ((0, 0, 0), 1)):
        reps = [n, H, Wp - (1 if origin[2] else 0)]
        tin = ((n, H, W), origin, [[1, 0, 0], [0, 1, 0], [0, 0, P]], [[0], [0], [1]], [P])
        tout = ((n, H, reps[2] * Q), (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, Q]], [[0], [0], [1]], [Q])
        store = torch.zeros(a.size + 16, dtype=torch.uint8, device="cuda")
        x = store[poff:poff + a.size].view(a.shape)
        x.copy_(torch.from_numpy(a))
        for D, B in ((1, 0), (6, 3), (1 << 20, 5)):
            want = oracle.run_task(a, oracle.make_tiler(*tin), tout[0], oracle.make_tiler(*tout), reps,
                                   oracle.make_stage(P, P, 0, w, D, B))
            y = torch.zeros(tout[0], dtype=torch.uint8, device="cuda")
            ds.run_task(x, ds.make_tiler(*tin), y, ds.make_tiler(*tout), reps,
                        ds.make_body(w, D, B, n_in=P))
            torch.cuda.synchronize()
            assert np.array_equal(y.cpu().numpy(), want), (origin, poff, D, B)


def _noclamp_body(rng, P, Q):
    """A body whose clamps can never fire (non-negative taps, bias in [0, D),
    D >= every output's tap sum, so 0 <= acc / D <= 255 and outputs reach 255):
    the kernels' host-proved noclamp branch.  D == 1 too (one unit tap)."""
    if rng.integers(0, 3) == 0:
        w = [[0] * P for _ in range(Q)]
        for k in range(Q):
            w[k][int(rng.integers(0, P))] = 1
        return w, 1, 0
    w = [[int(x) for x in rng.integers(0, 128, P)] for _ in range(Q)]
    D = max(1, max(sum(r) for r in w))
    return w, D, int(rng.integers(0, D))


@pytest.mark.gpu
def test_run_task_affine_columns():
    """Column-vector path: the innermost repetition dim is unit-stride in both
    arrays (extent % 4 == 0) and the pattern runs down a column, as in the
    paper's V task; 4 repetitions per thread, 4x4 byte transposes + dp4a."""
    rng = np.random.default_rng(fuzz_seed(99))
    for trial in range(40 * FUZZ_SCALE):
        P = int(rng.integers(1, 17))
        Q = int(rng.integers(1, 9))
        C = 4 * int(rng.integers(1, 40))                 # columns = innermost repetitions
        G = int(rng.integers(1, 12))                     # row groups
        S = int(rng.integers(1, P + 2))                  # row paving (overlapping windows when S < P)
        step = int(rng.choice([1, 2, -1]))               # pattern step down the column
        Hin = S * (G - 1) + abs(step) * (P - 1) + 1 + int(rng.integers(0, 5))
        o = abs(step) * (P - 1) if step < 0 else 0
        o += int(rng.integers(0, Hin - (S * (G - 1) + abs(step) * (P - 1))))
        three = trial % 4 == 0
        if three:
            F = int(rng.integers(1, 4))
            in_shape, out_shape = (F, Hin, C), (F, G * Q, C)
            tin = (in_shape, (0, o, 0), [[1, 0, 0], [0, S, 0], [0, 0, 1]], [[0], [step], [0]], [P])
            tout = (out_shape, (0, 0, 0), [[1, 0, 0], [0, Q, 0], [0, 0, 1]], [[0], [1], [0]], [Q])
            reps = [F, G, C]
        else:
            in_shape, out_shape = (Hin, C), (G * Q, C)
            tin = (in_shape, (o, 0), [[S, 0], [0, 1]], [[step], [0]], [P])
            tout = (out_shape, (0, 0), [[Q, 0], [0, 1]], [[1], [0]], [Q])
            reps = [G, C]
        if trial % 3 == 1:
            w, D, B = _noclamp_body(rng, P, Q)
        else:
            w = [[int(x) for x in rng.integers(-128, 128, P)] for _ in range(Q)]
            D = int(rng.choice([1, 3, 8, 999983]))
            B = int(rng.integers(-500, 500))
        a = rng.integers(0, 256, in_shape).astype(np.uint8)
        want = oracle.run_task(a, oracle.make_tiler(*tin), out_shape, oracle.make_tiler(*tout), reps,
                               oracle.make_stage(P, P, 0, w, D, B))
        y = torch.zeros(out_shape, dtype=torch.uint8, device="cuda")
        ds.run_task(torch.from_numpy(a).cuda(), ds.make_tiler(*tin), y, ds.make_tiler(*tout), reps,
                    ds.make_body(w, D, B, n_in=P))
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), want), (trial, P, Q, C, G, S, step, D)


@pytest.mark.gpu
@pytest.mark.parametrize("shift", [3, -2, 5, -7])
def test_run_task_peeled_wrap(shift):
    """Tilers that wrap only at one end of one repetition dimension (an H task
    whose column origin is shifted, a V task whose row origin is shifted) are
    split: the wrap-free interior on the fast paths, the thin slab on the
    modulo path -- the result must equal the oracle's modulo semantics."""
    rng = np.random.default_rng(100 + shift)
    n, H, W = 3, 18, 352
    a = rng.integers(0, 256, (n, H, W)).astype(np.uint8)
    hw = [[1, 5, 0, 0, 0, 0, 0, 0], [0, 0, 0, 3, 3, 0, 0, 0], [0, 0, 0, 0, 0, 0, 5, 1]]
    # H task, column origin shifted: the last (shift > 0) or first (< 0) window of a row wraps
    tin = ((n, H, W), (0, 0, shift), [[1, 0, 0], [0, 1, 0], [0, 0, 8]], [[0], [0], [1]], [8])
    tout = ((n, H, W // 8 * 3), (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, 3]], [[0], [0], [1]], [3])
    reps = [n, H, W // 8]
    want = oracle.run_task(a, oracle.make_tiler(*tin), tout[0], oracle.make_tiler(*tout), reps,
                           oracle.make_stage(8, 8, 0, hw, 6, 3))
    y = torch.zeros(tout[0], dtype=torch.uint8, device="cuda")
    ds.run_task(torch.from_numpy(a).cuda(), ds.make_tiler(*tin), y, ds.make_tiler(*tout), reps,
                ds.make_body(hw, 6, 3, n_in=8))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), want), "H task"
    # V task, row origin shifted: the last / first 9-row window wraps down the plane
    Wm = 132
    m = rng.integers(0, 256, (n, H, Wm)).astype(np.uint8)
    vw = [[3, 5, 0, 0, 0, 0, 0, 0, 0], [0, 0, 1, 7, 0, 0, 0, 0, 0], [0, 0, 0, 0, 0, 7, 1, 0, 0],
          [0, 0, 0, 0, 0, 0, 0, 5, 3]]
    tin = ((n, H, Wm), (0, shift, 0), [[1, 0, 0], [0, 9, 0], [0, 0, 1]], [[0], [1], [0]], [9])
    tout = ((n, H // 9 * 4, Wm), (0, 0, 0), [[1, 0, 0], [0, 4, 0], [0, 0, 1]], [[0], [1], [0]], [4])
    reps = [n, H // 9, Wm]
    want = oracle.run_task(m, oracle.make_tiler(*tin), tout[0], oracle.make_tiler(*tout), reps,
                           oracle.make_stage(9, 9, 0, vw, 8, 4))
    y = torch.zeros(tout[0], dtype=torch.uint8, device="cuda")
    ds.run_task(torch.from_numpy(m).cuda(), ds.make_tiler(*tin), y, ds.make_tiler(*tout), reps,
                ds.make_body(vw, 8, 4, n_in=9))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), want), "V task"


@pytest.mark.gpu
@pytest.mark.parametrize("P,Q", [(4, 1), (8, 3), (12, 5), (16, 8)])
def test_run_task_dense_large(P, Q):
    """Large dense tasks (11,100 repetitions: 86 full warps of 128 plus a
    ragged tail of 92) across pattern sizes 4-16 and 1-8 outputs, divisors on
    both sides of the exact multiply-high bound."""
    rng = np.random.default_rng(P * 10 + Q)
    n, H, Wp = 3, 37, 100                          # 11,100 repetitions
    W = P * Wp
    a = rng.integers(0, 256, (n, H, W)).astype(np.uint8)
    w = [[int(x) for x in rng.integers(-128, 128, P)] for _ in range(Q)]
    tin = ((n, H, W), (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, P]], [[0], [0], [1]], [P])
    tout = ((n, H, Wp * Q), (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, Q]], [[0], [0], [1]], [Q])
    reps = [n, H, Wp]
    bodies = [(w, D, B) for D, B in ((1, 0), (6, 3), (999983, 7))]
    bodies += [_noclamp_body(rng, P, Q) for _ in range(3)]
    for w, D, B in bodies:
        want = oracle.run_task(a, oracle.make_tiler(*tin), tout[0], oracle.make_tiler(*tout), reps,
                               oracle.make_stage(P, P, 0, w, D, B))
        y = torch.zeros(tout[0], dtype=torch.uint8, device="cuda")
        ds.run_task(torch.from_numpy(a).cuda(), ds.make_tiler(*tin), y, ds.make_tiler(*tout), reps,
                    ds.make_body(w, D, B, n_in=P))
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), want), (P, Q, D, B)

"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's golden vectors
and the pinned CPU oracle.  Indices bitwise; fp32 / fp64 means and gradients bitwise (the
north-star gate is 1e-5 relative, asserted in addition wherever bitwise is checked); bf16
bitwise against the bf16 rounding of the fp32 oracle on bf16-rounded inputs (gate 1e-2)."""

import numpy as np
import pytest
import torch

from conftest import iter_cases

pytestmark = pytest.mark.gpu

FP32_RTOL = 1e-5
BF16_RTOL = 1e-2


@pytest.fixture(scope="module")
def fsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_13645_b200 as m
    from paper_2511_13645_b200 import _lib
    _lib.load()
    return m


def dev_graph(fsa, rowptr, col, n):
    return fsa.CsrGraph.from_arrays(rowptr, col, device="cuda", num_nodes=n)


def T(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def bitwise(a: torch.Tensor, b: np.ndarray) -> bool:
    a = a.detach().cpu().numpy()
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def assert_close(got: torch.Tensor, want: np.ndarray, rtol):
    g = got.detach().double().cpu().numpy()
    w = want.astype(np.float64)
    np.testing.assert_allclose(g, w, rtol=rtol, atol=rtol * max(1.0, float(np.abs(w).max(initial=0))))


# ---- RNG / arithmetic hooks -----------------------------------------------------------------
def test_derive_states_hook(fsa, golden_rng):
    from paper_2511_13645_b200 import _lib
    g = golden_rng
    n = len(g["base"])
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    base = T(g["base"].view(np.int64))
    args = [T(g[k].astype(np.int64)) for k in ("root", "hop", "index")]
    _lib.check(_lib.load().fsa_derive_states(base.data_ptr(), *[a.data_ptr() for a in args], n,
                                             out.data_ptr(), torch.cuda.current_stream().cuda_stream), "derive")
    assert np.array_equal(out.cpu().numpy().view(np.uint64), g["derived"])


def test_xorshift_and_jump_hooks(fsa, golden_rng):
    from paper_2511_13645_b200 import _lib
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    g = golden_rng
    out = torch.empty(1000, dtype=torch.int64, device="cuda")
    _lib.check(lib.fsa_xorshift_steps(int(g["kernel_start"]), 1000, out.data_ptr(), st), "steps")
    assert np.array_equal(out.cpu().numpy().view(np.uint64), g["kernel_steps"])
    # jump-ahead equals serial steps (distances 1..1000 from the same start)
    n = 1000
    states = torch.full((n,), int(np.int64(g["kernel_start"].view(np.int64))), dtype=torch.int64, device="cuda")
    dist = torch.arange(1, n + 1, dtype=torch.int64, device="cuda")
    jumped = torch.empty(n, dtype=torch.int64, device="cuda")
    _lib.check(lib.fsa_jump(states.data_ptr(), dist.data_ptr(), n, jumped.data_ptr(), st), "jump")
    assert np.array_equal(jumped.cpu().numpy().view(np.uint64), g["kernel_steps"])


def test_barrett_hook(fsa):
    from paper_2511_13645_b200 import _lib
    rng = np.random.default_rng(9)
    n = 1 << 20
    x = rng.integers(0, 2**63, size=n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=n).astype(np.uint64)
    m = rng.integers(2, 2**30 + 1, size=n).astype(np.uint32)
    m[:64] = [2, 3, 4, 8, 16, 1 << 29, 1 << 30, (1 << 30) - 1] * 8
    x[:16] = np.iinfo(np.uint64).max
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    xd, md = T(x.view(np.int64)), T(m.view(np.int32))
    _lib.check(_lib.load().fsa_umod(xd.data_ptr(), md.data_ptr(), n, out.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream), "umod")
    assert np.array_equal(out.cpu().numpy().view(np.uint32), (x % m.astype(np.uint64)).astype(np.uint32))


# ---- golden forward / backward ----------------------------------------------------------------
@pytest.mark.parametrize("which", ["small", "powerlaw"])
def test_golden_cases(fsa, golden_small, golden_powerlaw, which):
    d = golden_small if which == "small" else golden_powerlaw
    for name, c in iter_cases(d):
        g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
        X = T(c["X"])
        seeds = T(c["seeds"])
        out1, i1 = fsa.fused_1hop_forward(g, X, seeds, c["k1"], c["base_seed"])
        assert bitwise(i1.samples, c["samples"]), name
        assert bitwise(i1.takes, c["takes"]), name
        assert bitwise(out1, c["out1"]), name
        out2, i2 = fsa.fused_2hop_forward(g, X, seeds, c["k1"], c["k2"], c["base_seed"])
        assert bitwise(i2.s1, c["s1"]), name
        assert bitwise(i2.s2, c["s2"]), name
        assert bitwise(out2, c["out2"]), name
        g1 = fsa.fused_1hop_backward(T(c["gout1"]), i1, c["N"])
        assert bitwise(g1, c["grad1"]), name
        g2 = fsa.fused_2hop_backward(T(c["gout2"]), i2, c["N"])
        assert bitwise(g2, c["grad2"]), name
        assert_close(g2, c["grad2"], FP32_RTOL)


def test_host_mode_numpy_in_numpy_out(fsa, golden_small):
    """Reference-style call: numpy arrays in, numpy arrays out (the graph as a plain object)."""
    class G:  # duck-typed reference CsrGraph
        pass

    for name, c in iter_cases(golden_small):
        g = G()
        g.num_nodes, g.rowptr, g.col = c["N"], c["rowptr"], c["col"]
        out2, idx = fsa.fused_2hop_forward(g, c["X"], c["seeds"], c["k1"], c["k2"], c["base_seed"])
        assert isinstance(out2, np.ndarray) and out2.tobytes() == c["out2"].tobytes(), name
        assert np.array_equal(idx.s2, c["s2"]), name
        grad = fsa.fused_2hop_backward(c["gout2"], idx, c["N"])
        assert isinstance(grad, np.ndarray) and grad.tobytes() == c["grad2"].tobytes(), name


def test_config1(fsa, golden_config1):
    c = golden_config1
    N, D, k, bs = (int(x) for x in c["meta"])
    X = np.random.default_rng([42, 1]).standard_normal((N, D)).astype(np.float32)
    g = dev_graph(fsa, c["rowptr"], c["col"], N)
    out, idx = fsa.fused_1hop_forward(g, T(X), T(c["seeds"]), k, bs)
    assert bitwise(idx.samples, c["samples"]) and bitwise(idx.takes, c["takes"])
    assert bitwise(out, c["out"])
    gout = np.random.default_rng(int(c["gout_seed"])).standard_normal(out.shape).astype(np.float32)
    grad = fsa.fused_1hop_backward(T(gout), idx, N).cpu().numpy()
    assert np.array_equal(np.nonzero(np.any(grad != 0, axis=1))[0], c["touched"])
    assert grad[c["touched"]].tobytes() == c["grad_rows"].tobytes()


# ---- semantics ------------------------------------------------------------------------------------
def test_nosave_identical_and_zero_backward(fsa, golden_powerlaw):
    for name, c in iter_cases(golden_powerlaw):
        g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
        X, seeds = T(c["X"]), T(c["seeds"])
        bare, none_idx = fsa.fused_2hop_forward(g, X, seeds, c["k1"], c["k2"], c["base_seed"], save_indices=False)
        assert none_idx is None and bitwise(bare, c["out2"])
        bare1, n1 = fsa.fused_1hop_forward(g, X, seeds, c["k1"], c["base_seed"], save_indices=False)
        assert n1 is None and bitwise(bare1, c["out1"])
        z = fsa.fused_2hop_backward(torch.ones_like(bare), None, c["N"])
        assert z.shape == (c["N"], X.shape[1]) and not bool(z.any())


def test_sampling_only_entry_points(fsa, golden_powerlaw):
    for name, c in iter_cases(golden_powerlaw):
        g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
        smp, tk = fsa.sample_1hop(g, T(c["seeds"]), c["k1"], c["base_seed"])
        assert bitwise(smp, c["samples"]) and bitwise(tk, c["takes"])
        s1, s2, t1, t2 = fsa.sample_2hop(g, T(c["seeds"]), c["k1"], c["k2"], c["base_seed"])
        assert bitwise(s1, c["s1"]) and bitwise(s2, c["s2"])
        assert np.array_equal(t1.cpu().numpy(), (c["s1"] >= 0).sum(1))
        assert np.array_equal(t2.cpu().numpy(), (c["s2"] >= 0).sum(2))


def test_errors_match_reference_messages(fsa):
    star = dev_graph(fsa, np.array([0, 3, 4, 5, 6]), np.array([1, 2, 3, 0, 0, 0]), 4)
    X = torch.zeros((4, 2), device="cuda", dtype=torch.float64)
    with pytest.raises(ValueError, match="seed out of range"):
        fsa.fused_1hop_forward(star, X, torch.tensor([17], device="cuda"), k=2, base_seed=0)
    with pytest.raises(ValueError, match="features must be"):
        fsa.fused_1hop_forward(star, torch.zeros((2, 2), device="cuda"), torch.tensor([0]), k=2, base_seed=0)
    with pytest.raises(ValueError, match="fanout"):
        fsa.fused_1hop_forward(star, X, torch.tensor([0]), k=0, base_seed=0)
    with pytest.raises(ValueError, match="fanouts"):
        fsa.fused_2hop_forward(star, X, torch.tensor([0]), 0, 2, base_seed=0)
    with pytest.raises(ValueError, match="seed batch"):
        fsa.fused_2hop_forward(star, X, torch.tensor([], dtype=torch.int64), 1, 2, base_seed=0)
    idx = fsa.SampledIndices1(samples=torch.tensor([[9]], dtype=torch.int32, device="cuda"),
                              takes=torch.tensor([1], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="out of range"):
        fsa.fused_1hop_backward(torch.ones((1, 1), device="cuda", dtype=torch.float64), idx, num_nodes=5)
    bad = fsa.SampledIndices1(samples=torch.tensor([[1]], dtype=torch.int32, device="cuda"),
                              takes=torch.tensor([-1], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="negative take"):
        fsa.fused_1hop_backward(torch.ones((1, 1), device="cuda", dtype=torch.float64), bad, num_nodes=5)
    i2 = fsa.SampledIndices2(s1=torch.tensor([[1, -1]], dtype=torch.int32, device="cuda"),
                             s2=torch.tensor([[[9, -1], [-1, -1]]], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="out of range"):
        fsa.fused_2hop_backward(torch.ones((1, 1), device="cuda"), i2, num_nodes=5)
    with pytest.raises(ValueError, match="batch size"):
        fsa.fused_2hop_backward(torch.ones((3, 1), device="cuda"), i2, num_nodes=50)


def test_device_error_flags_without_validation(fsa):
    from paper_2511_13645_b200 import _lib
    g = dev_graph(fsa, np.array([0, 1, 2]), np.array([1, 0]), 2)
    X = torch.ones((2, 4), device="cuda")
    fsa.device_errors()  # clear
    out, _ = fsa.fused_2hop_forward(g, X, torch.tensor([0, 5, 1], device="cuda"), 2, 2, 1, validate=False)
    assert fsa.device_errors() & _lib.FSA_DEVERR_SEED_RANGE
    assert fsa.device_errors() == 0


def test_backward_known_answers(fsa):
    # test_fused_1hop.py:87-109 and test_fused_2hop.py:70-78
    idx = fsa.SampledIndices1(samples=torch.tensor([[1, 2, -1]], dtype=torch.int32, device="cuda"),
                              takes=torch.tensor([2], dtype=torch.int32, device="cuda"))
    g = fsa.fused_1hop_backward(torch.tensor([[1.0]], device="cuda", dtype=torch.float64), idx, num_nodes=4)
    assert g[:, 0].tolist() == [0.0, 0.5, 0.5, 0.0]
    idx = fsa.SampledIndices1(samples=torch.tensor([[7, 3, -1, -1], [7, 1, 2, 5]], dtype=torch.int32, device="cuda"),
                              takes=torch.tensor([2, 4], dtype=torch.int32, device="cuda"))
    g = fsa.fused_1hop_backward(torch.tensor([[1.0], [1.0]], device="cuda", dtype=torch.float64), idx, num_nodes=8)
    assert float(g[7, 0]) == 0.75
    tree = dev_graph(fsa, np.array([0, 2, 3, 5, 5, 5, 5]), np.array([1, 2, 3, 4, 5]), 6)
    X = torch.tensor([[0.0], [0.0], [0.0], [1.0], [2.0], [4.0]], device="cuda", dtype=torch.float64)
    out, i2 = fsa.fused_2hop_forward(tree, X, torch.tensor([0], device="cuda"), 2, 2, 1)
    assert float(out[0, 0]) == 2.0
    gr = fsa.fused_2hop_backward(torch.tensor([[1.0]], device="cuda", dtype=torch.float64), i2, 6)
    assert gr[:, 0].tolist() == [0.0, 0.0, 0.0, 0.5, 0.25, 0.25]


def test_persistent_buffer_full_and_sparse_zeroing(fsa, golden_powerlaw):
    name, c = next(iter_cases(golden_powerlaw))
    g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
    X, seeds = T(c["X"]), T(c["seeds"])
    buf = torch.full((c["N"], X.shape[1]), 7.0, device="cuda")
    _, idx = fsa.fused_2hop_forward(g, X, seeds, c["k1"], c["k2"], c["base_seed"])
    r = fsa.fused_2hop_backward(T(c["gout2"]), idx, c["N"], out=buf)
    assert r is buf and bitwise(buf, c["grad2"])
    # a different batch through the sparse path must equal a fresh full computation
    seeds2 = torch.flip(seeds, [0])[:100]
    _, idx2 = fsa.fused_2hop_forward(g, X, seeds2, c["k1"], c["k2"], 99)
    go = torch.randn((100, X.shape[1]), device="cuda")
    fsa.fused_2hop_backward(T(c["gout2"]), idx, c["N"], out=buf, zero="sparse")
    fsa.fused_2hop_backward(go, idx2, c["N"], out=buf, zero="sparse")
    fresh = fsa.fused_2hop_backward(go, idx2, c["N"])
    assert torch.equal(buf, fresh)
    buf.add_(1.0)  # user modification -> version changes -> full fill next time
    fsa.fused_2hop_backward(go, idx2, c["N"], out=buf, zero="sparse")
    assert torch.equal(buf, fresh)


def test_sparse_coo_outputs(fsa, golden_powerlaw):
    for name, c in iter_cases(golden_powerlaw):
        g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
        _, idx = fsa.fused_2hop_forward(g, T(c["X"]), T(c["seeds"]), c["k1"], c["k2"], c["base_seed"])
        T2 = idx.s2.numel()
        touched = torch.empty(T2, dtype=torch.int32, device="cuda")
        nt = torch.empty(1, dtype=torch.int32, device="cuda")
        rows = torch.empty((T2, c["X"].shape[1]), device="cuda")
        dense = fsa.fused_2hop_backward(T(c["gout2"]), idx, c["N"], touched=touched, n_touched=nt, grad_rows=rows)
        n = int(nt)
        ids = touched[:n].long()
        assert n == len(np.unique(c["s2"][c["s2"] >= 0]))
        assert torch.equal(rows[:n], dense[ids])
        none = fsa.fused_2hop_backward(T(c["gout2"]), idx, c["N"], out=False, touched=touched, n_touched=nt,
                                       grad_rows=rows)
        assert none is None and int(nt) == n


# ---- dtypes --------------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_half_precision_features(fsa, oracle_mod, golden_powerlaw, dtype):
    for name, c in iter_cases(golden_powerlaw):
        g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
        Xh = T(c["X"]).to(dtype)
        Xr = Xh.float().cpu().numpy()  # the exact inputs the kernel sees
        out2, idx = fsa.fused_2hop_forward(g, Xh, T(c["seeds"]), c["k1"], c["k2"], c["base_seed"])
        ref, *_ = oracle_mod.fused_2hop(c["rowptr"], c["col"], Xr, c["seeds"], c["k1"], c["k2"], c["base_seed"])
        assert out2.dtype == dtype
        assert torch.equal(out2, torch.from_numpy(ref).cuda().to(dtype)), name  # fp32 acc, one rounding
        assert_close(out2.float(), ref, BF16_RTOL)
        gh = T(c["gout2"]).to(dtype)
        gr = fsa.fused_2hop_backward(gh, idx, c["N"])
        rg = oracle_mod.backward_2hop(gh.float().cpu().numpy(), c["s1"], c["s2"], c["N"])
        assert torch.equal(gr, torch.from_numpy(rg).cuda().to(dtype)), name


def test_padded_and_unaligned_rows(fsa, oracle_mod, golden_powerlaw):
    """Row strides that defeat 16-byte vectors (D=602-like widths) still match bitwise."""
    name, c = next(iter_cases(golden_powerlaw))
    g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
    for D, stride in ((13, 13), (6, 6), (10, 16), (3, 5)):
        base = torch.randn((c["N"], stride), device="cuda")
        X = base[:, :D]
        out, _ = fsa.fused_2hop_forward(g, X, T(c["seeds"]), c["k1"], c["k2"], c["base_seed"])
        ref, *_ = oracle_mod.fused_2hop(c["rowptr"], c["col"], X.contiguous().cpu().numpy(), c["seeds"],
                                        c["k1"], c["k2"], c["base_seed"])
        assert out.cpu().numpy().tobytes() == ref.tobytes(), (D, stride)


# ---- autograd ---------------------------------------------------------------------------------------
def test_autograd_function(fsa, golden_powerlaw):
    name, c = next(iter_cases(golden_powerlaw))
    g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
    X = T(c["X"]).requires_grad_(True)
    out, idx = fsa.fused_sample_agg_2hop(X, g, T(c["seeds"]), c["k1"], c["k2"], c["base_seed"])
    assert bitwise(out, c["out2"]) and bitwise(idx.s2, c["s2"])
    (out * T(c["gout2"])).sum().backward()
    assert bitwise(X.grad, c["grad2"])
    X.grad = None
    out, idx = fsa.fused_sample_agg_2hop(X, g, T(c["seeds"]), c["k1"], c["k2"], c["base_seed"], save_indices=False)
    out.sum().backward()
    assert idx is None and not bool(X.grad.any())
    X1 = T(c["X"]).requires_grad_(True)
    o1, i1 = fsa.fused_sample_agg_1hop(X1, g, T(c["seeds"]), c["k1"], c["base_seed"])
    (o1 * T(c["gout1"])).sum().backward()
    assert bitwise(X1.grad, c["grad1"])


def test_fd_gradient_fp64(fsa, golden_small):
    """Central finite differences at fp64 (test_fused_2hop.py:89-104)."""
    for name, c in list(iter_cases(golden_small))[:8]:
        if c["X"].dtype != np.float64:
            continue
        g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
        X = T(c["X"])
        seeds = T(c["seeds"])
        out, idx = fsa.fused_2hop_forward(g, X, seeds, c["k1"], c["k2"], c["base_seed"])
        w = T(np.random.default_rng(4).standard_normal(tuple(out.shape)))
        analytic = fsa.fused_2hop_backward(w, idx, c["N"]).cpu().numpy()
        eps = 1e-6
        fd = np.zeros_like(analytic)
        for v in range(c["N"]):
            for d in range(X.shape[1]):
                P = X.clone()
                P[v, d] += eps
                fp = float((w * fsa.fused_2hop_forward(g, P, seeds, c["k1"], c["k2"], c["base_seed"], False)[0]).sum())
                P[v, d] -= 2 * eps
                fm = float((w * fsa.fused_2hop_forward(g, P, seeds, c["k1"], c["k2"], c["base_seed"], False)[0]).sum())
                fd[v, d] = (fp - fm) / (2 * eps)
        # central differences at eps=1e-6 carry ~1e-10 absolute rounding noise in fp64, so the
        # relative gate of the reference (1e-6) is applied with a 1e-3 floor on the scale
        scale = np.maximum(np.abs(analytic), 1e-3)
        assert np.max(np.abs(fd - analytic) / scale) < 1e-6, name


# ---- determinism / sharding -------------------------------------------------------------------------
def test_repeat_and_shard_invariance(fsa, golden_powerlaw):
    for name, c in iter_cases(golden_powerlaw):
        g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
        X, seeds = T(c["X"]), T(c["seeds"])
        blobs = set()
        for _ in range(3):
            out, idx = fsa.fused_2hop_forward(g, X, seeds, c["k1"], c["k2"], c["base_seed"])
            gr = fsa.fused_2hop_backward(T(c["gout2"]), idx, c["N"])
            blobs.add(out.cpu().numpy().tobytes() + idx.s2.cpu().numpy().tobytes() + gr.cpu().numpy().tobytes())
        assert len(blobs) == 1
        B = seeds.numel()
        cuts = [0, 1, B // 4, B // 2 + 3, B]
        outs, s2s = [], []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            o, i = fsa.fused_2hop_forward(g, X, seeds[lo:hi], c["k1"], c["k2"], c["base_seed"], root_offset=lo)
            outs.append(o)
            s2s.append(i.s2)
        assert bitwise(torch.cat(outs), c["out2"]) and bitwise(torch.cat(s2s), c["s2"])


def test_division_hook(fsa):
    """The backward divides by a per-slot reciprocal (Markstein); it must equal IEEE division
    bitwise for every denominator the op can produce (max(t1,1)*max(t2,1) <= k1*k2)."""
    from paper_2511_13645_b200 import _lib
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().fsa_div_check(4096, bad.data_ptr(), torch.cuda.current_stream().cuda_stream), "div")
    torch.cuda.synchronize()
    assert int(bad.item()) == 0


def test_phase_entry_points_equal_monolithic_calls(fsa, golden_powerlaw):
    """fsa_fused_2hop_fwd_phase (SAMPLE, GATHER) and fsa_fused_2hop_bwd_phase (PLAN, TERMS, ROWS
    in any grouping), the split the step executor schedules across streams, give the monolithic
    calls' results bitwise."""
    from paper_2511_13645_b200 import _lib
    lib = _lib.load()
    name, c = next(iter_cases(golden_powerlaw))
    g = dev_graph(fsa, c["rowptr"], c["col"], c["N"])
    X, seeds = T(c["X"]), T(c["seeds"])
    B, k1, k2, D, N = seeds.numel(), c["k1"], c["k2"], X.shape[1], c["N"]
    ref_out, ref_idx = fsa.fused_2hop_forward(g, X, seeds, k1, k2, c["base_seed"])
    gout = torch.randn((B, D), device="cuda", dtype=X.dtype)
    ref_grad = fsa.fused_2hop_backward(gout, ref_idx, N)
    st = torch.cuda.current_stream().cuda_stream
    ws_f = torch.zeros(lib.fsa_ws_bytes(_lib.FSA_OP_FWD2, B, k1, k2, 0, 0, 0), dtype=torch.uint8, device="cuda")
    code = _lib.FSA_F32 if X.dtype == torch.float32 else _lib.FSA_F64
    ws_b = torch.zeros(lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, B, k1, k2, D, code, N), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(ref_out)
    s1 = torch.empty((B, k1), dtype=torch.int32, device="cuda")
    s2 = torch.empty((B, k1, k2), dtype=torch.int32, device="cuda")
    t1 = torch.empty(B, dtype=torch.int32, device="cuda")
    t2 = torch.empty((B, k1), dtype=torch.int32, device="cuda")
    for phase in (_lib.FSA_FWD_SAMPLE, _lib.FSA_FWD_GATHER):
        _lib.check(lib.fsa_fused_2hop_fwd_phase(
            g.rowptr.data_ptr(), g.col.data_ptr(), N, X.data_ptr(), D, X.stride(0), code, seeds.data_ptr(), B, 0,
            k1, k2, c["base_seed"] & (2**64 - 1), None, 1, s1.data_ptr(), s2.data_ptr(), t1.data_ptr(),
            t2.data_ptr(), out.data_ptr(), out.stride(0), ws_f.data_ptr(), ws_f.numel(), st, phase), "fwd phase")
    assert torch.equal(s1, ref_idx.s1) and torch.equal(s2, ref_idx.s2)
    assert torch.equal(out, ref_out)
    P, Tm, R = _lib.FSA_BWD_PLAN, _lib.FSA_BWD_TERMS, _lib.FSA_BWD_ROWS
    for split in ((P, _lib.FSA_BWD_APPLY), (P | Tm, R), (P, Tm, R), (Tm, P, R)):
        grad = torch.zeros((N, D), device="cuda", dtype=X.dtype)
        for phase in split:  # grad_out is only needed from TERMS on
            _lib.check(lib.fsa_fused_2hop_bwd_phase(
                gout.data_ptr() if phase & Tm else None, B, D, D, code, s1.data_ptr(), s2.data_ptr(), k1, k2, N,
                grad.data_ptr(), 0, None, None, None, ws_b.data_ptr(), ws_b.numel(), st, phase), "bwd phase")
        torch.cuda.synchronize()
        assert torch.equal(grad, ref_grad), split
    with pytest.raises(RuntimeError):  # TERMS without grad_out
        _lib.check(lib.fsa_fused_2hop_bwd_phase(
            None, B, D, D, code, s1.data_ptr(), s2.data_ptr(), k1, k2, N, grad.data_ptr(), 0, None, None, None,
            ws_b.data_ptr(), ws_b.numel(), st, Tm), "bwd phase")


@pytest.mark.parametrize("B,leaves", [(40, 64), (1024, 3000)])
def test_hub_hit_by_every_slot(fsa, oracle_mod, B, leaves):
    """A star graph whose roots are all the centre: every second-hop slot samples the centre, so
    the replay backward sums B * k1 terms into one row (k_bwd_big: counting sort at 600 hits,
    bitmap windows at 15 360) — bitwise against the oracle."""
    n = leaves + 1
    rowptr = np.zeros(n + 1, np.int64)
    rowptr[1] = leaves
    rowptr[2:] = leaves + np.arange(1, leaves + 1)
    col = np.concatenate([np.arange(1, n), np.zeros(leaves, np.int64)]).astype(np.int32)
    g = dev_graph(fsa, rowptr, col, n)
    rng = np.random.default_rng(11)
    X = rng.standard_normal((n, 40)).astype(np.float32)
    seeds = np.zeros(B, np.int64)
    k1, k2, bs = 15, 10, 1234567
    out, idx = fsa.fused_2hop_forward(g, T(X), T(seeds), k1, k2, bs)
    gout = rng.standard_normal((B, 40)).astype(np.float32)
    grad = fsa.fused_2hop_backward(T(gout), idx, n)
    torch.cuda.synchronize()
    ref_out, s1, s2, _, _ = oracle_mod.fused_2hop(rowptr.astype(np.int32), col, X, seeds, k1, k2, bs)
    ref_grad = oracle_mod.backward_2hop(gout, s1, s2, n)
    assert int((s2 == 0).sum()) == B * k1
    assert np.array_equal(idx.s2.cpu().numpy(), s2)
    assert bitwise(out, ref_out)
    assert bitwise(grad, ref_grad)


@pytest.mark.parametrize("D,dtype", [(300, torch.float32), (602, torch.bfloat16), (37, torch.float64),
                                     (130, torch.float16)])
def test_wide_rows_dense_collisions(fsa, oracle_mod, D, dtype):
    """A small random graph with wide rows: most second-hop nodes are hit several times, so
    every row writer runs on rows wider than one warp's chunk span (the multi-hit kernel's wide
    path, many term-table chunks per group), with dense and COO outputs — bitwise against the
    oracle on the same (rounded) inputs."""
    rng = np.random.default_rng(D)
    n, deg = 3000, 40  # every row also lists node 0: a hub next to ~13-hit ordinary nodes
    col = np.stack([np.concatenate([[0], np.sort(rng.choice(np.arange(1, n), deg - 1, replace=False))])
                    for _ in range(n)]).astype(np.int32).ravel()
    rowptr = np.arange(0, n * deg + 1, deg, dtype=np.int64)
    g = dev_graph(fsa, rowptr, col, n)
    Xd = T(rng.standard_normal((n, D)).astype(np.float32)).to(dtype)
    seeds = rng.integers(0, n, 256).astype(np.int64)
    k1, k2, bs = 15, 10, 987654321
    out, idx = fsa.fused_2hop_forward(g, Xd, T(seeds), k1, k2, bs)
    gout = T(rng.standard_normal((256, D)).astype(np.float32)).to(dtype)
    T2 = idx.s2.numel()
    touched = torch.empty(T2, dtype=torch.int32, device="cuda")
    nt = torch.empty(1, dtype=torch.int32, device="cuda")
    rows = torch.empty((T2, D), device="cuda", dtype=dtype)
    grad = fsa.fused_2hop_backward(gout, idx, n, touched=touched, n_touched=nt, grad_rows=rows)
    torch.cuda.synchronize()
    acc = np.float64 if dtype == torch.float64 else np.float32
    ref_out, s1, s2, _, _ = oracle_mod.fused_2hop(rowptr.astype(np.int32), col, Xd.to(torch.float64).cpu().numpy().astype(acc),
                                                  seeds, k1, k2, bs)
    ref_grad = oracle_mod.backward_2hop(gout.to(torch.float64).cpu().numpy().astype(acc), s1, s2, n)
    assert np.array_equal(idx.s2.cpu().numpy(), s2)
    hits = np.bincount(s2[s2 >= 0], minlength=n)
    assert (hits > 1).sum() > 100 and hits.max() > 32  # multi-hit and hub paths both exercised
    assert torch.equal(out, torch.from_numpy(ref_out).cuda().to(dtype))
    want = torch.from_numpy(ref_grad).cuda().to(dtype)
    bad = (grad != want).any(1).nonzero().flatten().tolist()
    assert not bad, (bad[:8], hits[bad[:8]].tolist())
    k = int(nt)
    assert k == int((hits > 0).sum())
    assert torch.equal(rows[:k], grad[touched[:k].long()])


def test_draw_loop_benchmark_hook(fsa):
    """fsa_bench_draws (the sampler's integer roofline, tools/bench_draws.py): one warp reports
    clock cycles, a grid of CTAs runs and can be timed; bad geometries are argument errors."""
    from paper_2511_13645_b200 import _lib
    lib = _lib.load()
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for mode in range(4):
        _lib.check(lib.fsa_bench_draws(mode, 1024, 20000, 10, 32, out.data_ptr(), st), "one warp")
        torch.cuda.synchronize()
        assert 0 < int(out[0]) < 1024 * 10_000  # cycles for 1,024 draws per lane
        _lib.check(lib.fsa_bench_draws(mode, 512, 20000, 10, 148 * 256, out.data_ptr(), st), "grid")
        torch.cuda.synchronize()
    assert lib.fsa_bench_draws(0, 1000, 20000, 10, 32, out.data_ptr(), st) == _lib.FSA_ERR_ARG  # n % 256
    assert lib.fsa_bench_draws(0, 512, 20000, 10, 300, out.data_ptr(), st) == _lib.FSA_ERR_ARG  # lanes % 256

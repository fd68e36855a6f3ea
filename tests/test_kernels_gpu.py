"""Kernel-level numerics: the tcgen05 GEMM (1-CTA and CTA-pair kernels) and
the fp32 SIMT GEMM, with every fused epilogue the engine uses, against a
plain PyTorch fp32 reference of the same op on the same (bf16-rounded)
inputs. Called through the C-ABI test hook orx_debug_gemm on device pointers.

Tolerances: fp32 outputs differ from torch only by accumulation order
(<= 1e-4 of the row's max magnitude); bf16 outputs add one bf16 rounding
(2^-8 relative).
"""
import ctypes as C

import numpy as np

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _lib():
    from paper_2506_13695_b200 import _lib
    return _lib


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def run_gemm(A, B, *, out, bias=None, row_scale=None, resid=None, row_map=None, act=0, swiglu=0, n_out=0,
             m_valid=0, col_off=0, tile_expert=None, n_mtiles=None, b_rows_per_expert=0, n_groups=0, tile_rows=0,
             force_single_cta=0, precision=1, sync=True):
    L = _lib()
    a = L.orx_gemm_args()
    a.A, a.lda = _ptr(A), A.stride(0)
    a.B, a.ldb = _ptr(B), B.stride(0)
    a.M, a.K = A.shape[0], A.shape[1]
    a.N = B.shape[0] if tile_expert is None else b_rows_per_expert
    a.precision = precision
    a.bias, a.row_scale, a.row_map = _ptr(bias), _ptr(row_scale), _ptr(row_map)
    a.resid, a.ld_resid = _ptr(resid), (resid.stride(0) if resid is not None else 0)
    a.out, a.ldo, a.out_bf16 = _ptr(out), out.stride(0), int(out.dtype == torch.bfloat16)
    a.act, a.swiglu, a.n_out, a.m_valid, a.col_off = act, swiglu, n_out, m_valid, col_off
    a.tile_expert, a.n_mtiles = _ptr(tile_expert), _ptr(n_mtiles)
    a.b_rows_per_expert, a.n_groups, a.tile_rows = b_rows_per_expert, n_groups, tile_rows
    a.force_single_cta = force_single_cta
    L.check(L.lib().orx_debug_gemm(C.byref(a), None))
    if sync:
        torch.cuda.synchronize()


def _act(x, act):
    if act == 1:
        return torch.where(x > 0, x, 0.01 * x)
    if act == 2:
        return x * torch.sigmoid(x)
    return x


def _close(got, want, bf16):
    scale = want.abs().amax(dim=-1, keepdim=True).clamp_min(1e-6)
    err = ((got.float() - want) / scale).abs().max().item()
    tol = 1.2e-2 if bf16 else 1e-4
    assert err <= tol, f"max row-relative error {err:.3e} > {tol:.1e}"
    return err


def _inputs(M, N, K, seed=0, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = (torch.rand(M, K, device="cuda", generator=g) - 0.5).to(dtype)
    B = ((torch.rand(N, K, device="cuda", generator=g) - 0.5) / K ** 0.5).to(dtype)
    return A, B


DENSE = [
    # (M, N, K, act, bias, out_bf16, resid)
    (1000, 1024, 2176, 1, True, True, False),   # lifelong fc1: LeakyReLU + bias, M not a multiple of 256
    (300, 1000, 200, 0, True, False, True),     # N / K tails, fp32 out + residual
    (4096, 3072, 1024, 0, False, True, False),  # fused QKV
    (128, 8192, 1024, 0, False, False, False),  # 1-CTA kernel (M <= 128): position head
    (2048, 2048, 1024, 2, True, True, False),   # FFN fc1: SiLU + bias
    (6000, 1024, 2048, 0, True, False, True),   # FFN fc2 + residual (fp32 stream)
    (1000, 128, 256, 1, True, True, False),     # BN=128 CTA-pair kernel
    (77, 96, 40, 0, True, False, True),         # tiny, 1-CTA BN=128
    (100, 1024, 1024, 0, True, False, True),    # M <= 128, N >= 512: 1-CTA BN=64 (decoder step 0), residual
    (64, 2048, 512, 2, True, True, False),      # same kernel, SiLU + bf16 out
]


@pytest.mark.parametrize("M,N,K,act,bias,out_bf16,resid", DENSE)
def test_gemm_dense(M, N, K, act, bias, out_bf16, resid):
    A, B = _inputs(M, N, K, seed=M + N + K)
    b = torch.linspace(-0.5, 0.5, N, device="cuda") if bias else None
    R = torch.randn(M, N, device="cuda") if resid else None
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if out_bf16 else torch.float32)
    run_gemm(A, B, out=out, bias=b, resid=R, act=act)
    want = A.float() @ B.float().t()
    if bias:
        want = want + b
    want = _act(want, act)
    if resid:
        want = want + R
    _close(out, want, out_bf16)


def test_gemm_pair_equals_single_cta():
    """The CTA-pair and 1-CTA tcgen05 kernels accumulate in the same order."""
    A, B = _inputs(1536, 2048, 1024, seed=7)
    o1 = torch.empty(1536, 2048, device="cuda")
    o2 = torch.empty_like(o1)
    run_gemm(A, B, out=o1)
    run_gemm(A, B, out=o2, force_single_cta=1)
    assert torch.equal(o1, o2)


def test_gemm_row_map_scale_resid():
    """Scatter epilogue: output row = row_map[r] (-1 dropped), per-row scale, residual."""
    M, N, K = 700, 1024, 512
    A, B = _inputs(M, N, K, seed=3)
    perm = torch.randperm(2 * M, device="cuda")[:M].to(torch.int32)
    perm[::7] = -1
    rs = torch.rand(M, device="cuda") + 0.5
    out = torch.randn(2 * M, N, device="cuda")
    base = out.clone()
    run_gemm(A, B, out=out, row_map=perm, row_scale=rs, resid=out)
    want = base.clone()
    keep = perm >= 0
    y = (A.float() @ B.float().t()) * rs[:, None]
    want[perm[keep].long()] = base[perm[keep].long()] + y[keep]
    _close(out, want, False)


@pytest.mark.parametrize("scale", [False, True])
def test_gemm_staged_row_map(scale):
    """Coalesced (SMEM-transposed) epilogue with scattered / dropped output rows:
    row_map + residual (specialised mode) and row_map + row scale, ragged M."""
    M, N, K = 777, 512, 256
    A, B = _inputs(M, N, K, seed=11)
    perm = torch.randperm(3 * M, device="cuda")[:M].to(torch.int32)
    perm[5::9] = -1
    out = torch.randn(3 * M, N, device="cuda")
    base = out.clone()
    rs = torch.rand(M, device="cuda") + 0.5 if scale else None
    run_gemm(A, B, out=out, row_map=perm, row_scale=rs, resid=None if scale else out)
    y = A.float() @ B.float().t()
    if scale:
        y = y * rs[:, None]
    want = base.clone()
    keep = perm >= 0
    want[perm[keep].long()] = (0 if scale else base[perm[keep].long()]) + y[keep]
    _close(out, want, False)


def _grouped_case(E, counts, h, d, tile_rows, seed):
    """Expert segments padded to tile_rows (moe_plan_kernel layout)."""
    segs, tiles, off = [], [], 0
    for e, c in enumerate(counts):
        nt = (c + tile_rows - 1) // tile_rows
        segs.append((off, c))
        tiles += [e] * nt
        off += nt * tile_rows
    S = off + tile_rows
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = torch.zeros(S, d, device="cuda", dtype=torch.bfloat16)
    for (o, c) in segs:
        X[o:o + c] = (torch.rand(c, d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    W1 = ((torch.rand(E, h, d, device="cuda", generator=g) - 0.5) / d ** 0.5).to(torch.bfloat16)
    W3 = ((torch.rand(E, h, d, device="cuda", generator=g) - 0.5) / d ** 0.5).to(torch.bfloat16)
    # interleave per 128 output columns: [W1 block | W3 block] per 256 rows (engine pack_moe)
    W13 = torch.empty(E, 2 * h, d, device="cuda", dtype=torch.bfloat16)
    for j in range(0, h, 128):
        W13[:, 2 * j:2 * j + 128] = W1[:, j:j + 128]
        W13[:, 2 * j + 128:2 * j + 256] = W3[:, j:j + 128]
    te = torch.full((S // tile_rows + 1,), -1, device="cuda", dtype=torch.int32)
    te[:len(tiles)] = torch.tensor(tiles, dtype=torch.int32)
    nmt = torch.tensor([len(tiles)], device="cuda", dtype=torch.int32)
    return segs, S, X, W1, W3, W13.reshape(E * 2 * h, d), te, nmt


@pytest.mark.parametrize("tile_rows", [256, 128])
def test_gemm_grouped_swiglu_and_combine(tile_rows):
    """MoE expert GEMMs: W1|W3 with the SwiGLU epilogue, then W2 with the gate weight as row scale."""
    E, h, d = 5, 384, 256
    counts = [300, 0, 17, 513, 256]
    segs, S, X, W1, W3, W13, te, nmt = _grouped_case(E, counts, h, d, tile_rows, seed=11)
    H = torch.zeros(S, h, device="cuda", dtype=torch.bfloat16)
    run_gemm(X, W13, out=H, swiglu=1, n_out=h, m_valid=S, tile_expert=te, n_mtiles=nmt,
             b_rows_per_expert=2 * h, n_groups=E, tile_rows=tile_rows, force_single_cta=int(tile_rows == 128))
    W2 = ((torch.rand(E, d, h, device="cuda") - 0.5) / h ** 0.5).to(torch.bfloat16)
    rs = torch.rand(S, device="cuda")
    Y = torch.zeros(S, d, device="cuda")
    run_gemm(H, W2.reshape(E * d, h), out=Y, row_scale=rs, n_out=d, m_valid=S, tile_expert=te, n_mtiles=nmt,
             b_rows_per_expert=d, n_groups=E, tile_rows=tile_rows)
    for e, (o, c) in enumerate(segs):
        if c == 0:
            continue
        x = X[o:o + c].float()
        a = x @ W1[e].float().t()
        b = x @ W3[e].float().t()
        hw = a * torch.sigmoid(a) * b
        _close(H[o:o + c], hw, True)
        yw = (H[o:o + c].float() @ W2[e].float().t()) * rs[o:o + c, None]
        _close(Y[o:o + c], yw, False)


@pytest.mark.parametrize("M,N,K", [(300, 1000, 200), (1024, 512, 384)])
def test_gemm_fp32_simt(M, N, K):
    """fp32 parity-mode GEMM (SIMT FFMA) with bias + SiLU + residual."""
    A, B = _inputs(M, N, K, seed=5, dtype=torch.float32)
    b = torch.randn(N, device="cuda")
    R = torch.randn(M, N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    run_gemm(A, B, out=out, bias=b, resid=R, act=2, precision=0)
    want = _act(A @ B.t() + b, 2) + R
    _close(out, want, False)


def _ref_topk_keys(logits, pscore, plex, k, lse):
    """torch restatement of the candidate key (beam.cuh) and its top-k set,
    on the kernel's own log-normaliser (so fp32 rounding of lse cannot reorder)."""
    V = logits.shape[1]
    sc = (pscore[:, None] + (logits - lse[:, None])).contiguous()
    bits = sc.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    neg = bits >= 0x80000000
    ordb = torch.where(neg, (~bits) & 0xFFFFFFFF, bits | 0x80000000)
    low = 0xFFFFFFFF - (plex[:, None].to(torch.int64) * V + torch.arange(V, device=logits.device))
    keys = (ordb << 32) | low  # unsigned order; flip the top bit for a signed torch sort
    skeys = keys ^ (-(1 << 63))
    return torch.topk(skeys, k, dim=1).values


@pytest.mark.parametrize("V,k,ties", [(8192, 128, False), (8192, 512, False), (8192, 32, False), (1000, 100, False),
                                      (8192, 128, True), (64, 16, False)])
def test_row_topk(V, k, ties):
    """Per-row log-softmax + top-k candidate keys (fast bisection path and the
    radix fallback taken under massive exact ties) vs a torch restatement."""
    rows = 300
    g = torch.Generator(device="cuda").manual_seed(V + k)
    logits = torch.randn(rows, V, device="cuda", generator=g) * 7.0
    if ties:
        logits = torch.round(logits / 8.0) * 8.0  # a handful of distinct values per row
    pscore = torch.randn(rows, device="cuda", generator=g) * 3.0
    plex = torch.randint(0, 100, (rows,), device="cuda", dtype=torch.int32, generator=g)
    lse = torch.empty(rows, device="cuda")
    cand = torch.empty(rows, k, device="cuda", dtype=torch.int64)
    L = _lib()
    L.lib().orx_debug_topk_fallback_rows()
    L.check(L.lib().orx_debug_row_topk(rows, V, k, _ptr(logits), _ptr(pscore), _ptr(plex), _ptr(lse), _ptr(cand),
                                       None))
    torch.cuda.synchronize()
    fallbacks = L.lib().orx_debug_topk_fallback_rows()
    print(f"V={V} k={k} ties={ties}: {fallbacks}/{rows} rows took the radix fallback")
    if ties:
        assert fallbacks > 0  # the exact-tie path is exercised
    elif V == 8192 and k <= 512:
        assert fallbacks <= rows // 20  # the fast path handles ordinary rows
    assert torch.allclose(lse, torch.logsumexp(logits, dim=1), rtol=1e-5, atol=1e-4)
    want_top = _ref_topk_keys(logits, pscore, plex, k, lse)
    got = torch.sort(cand ^ (-(1 << 63)), dim=1, descending=True).values
    assert torch.equal(got, want_top)


def _attn_case(kind, H=2, dh=128, seed=0):
    """(Q, K, V buffers, segment arrays, Vt) for the three attention uses of the hot path."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    d = H * dh
    rnd = lambda *s: (torch.randn(*s, device="cuda", generator=g)).to(torch.bfloat16)  # noqa: E731
    if kind == "encoder":  # self-attention over T=405 rows per user, fused QKV buffer (policy.cpp:261)
        B, T = 3, 405
        qkv = rnd(B * T, 3 * d)
        Q, K, V = qkv, qkv, qkv
        cols = (0, d, 2 * d)
        qs = [(b * T, T) for b in range(B)]
        ks = qs
    elif kind == "qformer":  # 128 shared learned queries over ragged lifelong keys (nn.cpp:97-100)
        klens = [2000, 1, 37]
        B = len(klens)
        Q = rnd(128, d)
        kv = rnd(sum(klens), 2 * d)
        K, V = kv, kv
        cols = (0, 0, d)
        starts = np.concatenate([[0], np.cumsum(klens)[:-1]])
        qs = [(0, 128)] * B
        ks = list(zip(starts.tolist(), klens))
    else:  # decoder cross-attention: W=128 beam rows of a user over its 405 encoder rows (policy.cpp:284)
        B, T, Wb = 2, 405, 128
        Q = rnd(B * Wb, d)
        kv = rnd(B * T, 2 * d)
        K, V = kv, kv
        cols = (0, 0, d)
        qs = [(b * Wb, Wb) for b in range(B)]
        ks = [(b * T, T) for b in range(B)]
    Lmax = max(k for _, k in ks)
    ld = (Lmax + 7) // 8 * 8
    Vt = torch.zeros(B * H * dh, ld, device="cuda", dtype=torch.bfloat16)
    for b, (s0, n) in enumerate(ks):
        for h in range(H):
            Vt[(b * H + h) * dh:(b * H + h + 1) * dh, :n] = V[s0:s0 + n, cols[2] + h * dh:cols[2] + (h + 1) * dh].t()
    return B, H, dh, Q, K, V, cols, qs, ks, Vt


@pytest.mark.parametrize("kind", ["encoder", "qformer", "cross"])
@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("dh", [32, 64, 128])
def test_attention_bf16(kind, kernel, dh):
    """Segmented softmax(QK^T/sqrt(dh))V (mha_core, tape.cpp:822-905): the
    mma.sync kernel (0) and the tcgen05/TMEM kernel (1, transposed V; 64-byte
    swizzled Q/K rows at dh=32, the 0.015B config) vs torch fp32."""
    B, H, dh, Q, K, V, cols, qs, ks, Vt = _attn_case(kind, H=256 // dh, dh=dh)
    d = H * dh
    rows_out = sum(n for _, n in qs)
    O = torch.zeros(rows_out, d, device="cuda", dtype=torch.bfloat16)
    ost = np.concatenate([[0], np.cumsum([n for _, n in qs])[:-1]])
    i32 = lambda xs: torch.tensor(xs, device="cuda", dtype=torch.int32)  # noqa: E731
    qst, qln = i32([s for s, _ in qs]), i32([n for _, n in qs])
    kst, kln = i32([s for s, _ in ks]), i32([n for _, n in ks])
    ostt = i32(ost.tolist())
    L = _lib()
    a = L.orx_attn_args()
    a.B, a.max_q, a.heads, a.dh = B, max(n for _, n in qs), H, dh
    a.Q, a.q_rows, a.ldq, a.q_col0 = _ptr(Q), Q.shape[0], Q.stride(0), cols[0]
    a.K, a.k_rows, a.ldk, a.k_col0 = _ptr(K), K.shape[0], K.stride(0), cols[1]
    a.V, a.ldv, a.v_col0 = _ptr(V), V.stride(0), cols[2]
    a.Vt, a.vt_rows, a.vt_cols, a.vt_ld = _ptr(Vt), Vt.shape[0], Vt.shape[1], Vt.stride(0)
    a.O, a.ldo = _ptr(O), O.stride(0)
    a.q_start, a.q_len, a.k_start, a.k_len, a.o_start = _ptr(qst), _ptr(qln), _ptr(kst), _ptr(kln), _ptr(ostt)
    a.kernel = kernel
    L.check(L.lib().orx_debug_attention(C.byref(a), None))
    torch.cuda.synchronize()
    assert torch.isfinite(O.float()).all(), "non-finite attention output"
    worst = 0.0
    for b in range(B):
        (q0, nq), (k0, nk) = qs[b], ks[b]
        for h in range(H):
            q = Q[q0:q0 + nq, cols[0] + h * dh:cols[0] + (h + 1) * dh].float()
            k = K[k0:k0 + nk, cols[1] + h * dh:cols[1] + (h + 1) * dh].float()
            v = V[k0:k0 + nk, cols[2] + h * dh:cols[2] + (h + 1) * dh].float()
            ref = torch.softmax(q @ k.t() / dh ** 0.5, dim=-1) @ v
            got = O[ost[b]:ost[b] + nq, h * dh:(h + 1) * dh].float()
            err = ((got - ref).abs().max() / ref.abs().max().clamp_min(1e-6)).item()
            assert err == err, "NaN error"
            worst = max(worst, err)
    print(f"attention {kind} kernel {kernel} dh={dh}: max rel err {worst:.3e}")
    assert worst < 3e-2

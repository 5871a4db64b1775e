"""Per-kernel parity on the B200: each CUDA kernel (through the C ABI, elis_ops.h)
against the oracle's per-op function on the same (bf16-representable) inputs.

Tolerances are derived from the arithmetic:
  * GEMM, bf16 out: fp32 accumulation then one bf16 rounding (rel 2^-8 = 3.9e-3);
  * GEMM, fp32 out (+ residual): fp32 accumulation of K bf16 products (~K * 2^-24 rel);
  * attention: P rounded to bf16 for the PV product, output rounded to bf16;
  * LayerNorm / FC head: pure fp32.
"""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def bf16_tensor(x: np.ndarray):
    """bf16-representable fp32 numpy -> (torch bf16 on cuda, exact fp64 numpy copy)."""
    x = inputs.round_to_bf16(np.asarray(x, np.float32))
    return torch.from_numpy(x).to(torch.bfloat16).cuda(), x.astype(np.float64)


def fp16_tensor(x: np.ndarray):
    """fp16-representable fp32 numpy -> (torch fp16 on cuda, exact fp64 numpy copy)."""
    t = torch.from_numpy(np.asarray(x, np.float32)).to(torch.float16)
    return t.cuda(), t.float().numpy().astype(np.float64)


def to_np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def attn_layout(qkv, H, nh):
    """qkv [T, 3H] -> the layout elis_op_attention expects: head-major planes [3 nh][T][64] for
    d = 64 (what the QKV GEMM writes), unchanged [T, 3H] for d = 32."""
    d = H // nh
    if d != 64:
        return qkv
    T = qkv.shape[0]
    return qkv.view(T, 3, nh, d).permute(1, 2, 0, 3).contiguous()


@pytest.mark.parametrize("M", [1, 129, 300, 1000])
@pytest.mark.parametrize("N,K", [(384, 128), (128, 128), (512, 128), (2304, 768), (768, 768), (3072, 768),
                                 (768, 3072), (1024, 1024)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_tcgen05_parity(cuda_lib, M, N, K, epi):
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    rng = np.random.default_rng(M * 7 + N + K + epi)
    A, A64 = bf16_tensor(rng.normal(0, 1, (M, K)))
    W, W64 = bf16_tensor(rng.normal(0, 0.05, (N, K)))
    b64 = rng.normal(0, 0.1, N).astype(np.float32)
    bias = torch.from_numpy(b64).cuda()
    ref = oenc.linear(A64, W64, b64.astype(np.float64))
    if epi == 0:
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        binding.op_gemm(A, W, bias, out, epi)
        torch.cuda.synchronize()
        got = to_np(out)
        assert np.abs(got - ref).max() <= 4e-3 * np.abs(ref).max() + 1e-6
        np.testing.assert_allclose(got, ref, rtol=8e-3, atol=2e-3)
    elif epi == 1:
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        binding.op_gemm(A, W, bias, out, epi)
        torch.cuda.synchronize()
        ref = oenc.gelu(ref)
        np.testing.assert_allclose(to_np(out), ref, rtol=8e-3, atol=2e-3)
    else:
        res64 = rng.normal(0, 1, (M, N)).astype(np.float32)
        res = torch.from_numpy(res64).cuda()
        out = torch.empty(M, N, dtype=torch.float32, device="cuda")
        binding.op_gemm(A, W, bias, out, epi, residual=res)
        torch.cuda.synchronize()
        ref = ref + res64.astype(np.float64)
        np.testing.assert_allclose(to_np(out), ref, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("M", [1, 129, 300, 1000, 4099])
@pytest.mark.parametrize("N,K,epi,hm", [(2304, 768, 0, True), (2304, 768, 0, False), (3072, 768, 1, False),
                                        (3072, 1024, 0, True), (4096, 1024, 1, False)])
def test_gemm_f16_parity(cuda_lib, M, N, K, epi, hm):
    """The fp16 instantiations the bench runs (QKV with the head-major store, FFN1 + GELU): fp32
    accumulation then one fp16 rounding of the output (rel 2^-11 = 4.9e-4)."""
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    rng = np.random.default_rng(M * 3 + N + K + epi)
    A, A64 = fp16_tensor(rng.normal(0, 1, (M, K)))
    W, W64 = fp16_tensor(rng.normal(0, 0.05, (N, K)))
    b64 = rng.normal(0, 0.1, N).astype(np.float32)
    ref = oenc.linear(A64, W64, b64.astype(np.float64))
    if epi == 1:
        ref = oenc.gelu(ref)
    out = torch.full((M * N,), float("nan"), dtype=torch.float16, device="cuda")
    binding.op_gemm_f16(A, W, torch.from_numpy(b64).cuda(), out, epi, head_major=hm)
    torch.cuda.synchronize()
    got = to_np(out)
    got = got.reshape(N // 64, M, 64).transpose(1, 0, 2).reshape(M, N) if hm else got.reshape(M, N)
    np.testing.assert_allclose(got, ref, rtol=2e-3, atol=5e-4 if epi == 0 else 8e-4)


@pytest.mark.parametrize("d,nh", [(64, 12), (32, 4), (64, 16)])
def test_attention_varlen_parity(cuda_lib, d, nh):
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    H = d * nh
    lengths = np.array([1, 2, 63, 64, 65, 130, 7, 512, 200, 33], dtype=np.int32)
    T = int(lengths.sum())
    rng = np.random.default_rng(d + nh)
    qkv, qkv64 = bf16_tensor(rng.normal(0, 1.0, (T, 3 * H)))
    ctx = torch.full((T, H), float("nan"), dtype=torch.bfloat16, device="cuda")
    lt = torch.from_numpy(lengths).cuda()
    binding.op_attention(attn_layout(qkv, H, nh), lt, H, nh, ctx)
    torch.cuda.synchronize()
    got = to_np(ctx)
    starts = inputs.offsets(lengths)
    for i, L in enumerate(lengths):
        sl = slice(starts[i], starts[i + 1])
        ref = oenc.attention(qkv64[sl, :H], qkv64[sl, H:2 * H], qkv64[sl, 2 * H:], nh)
        err = np.abs(got[sl] - ref).max()
        assert err < 2e-2, (i, int(L), err)


# lengths that exercise the packed short-request tiles (several requests of <= 128 tokens per
# 128-row tile in 32-row segments, segment tails, a full pack of four 1..32-token requests) next to
# long requests with a partial last q tile / key block
PACK_LENGTHS = [1, 2, 31, 32, 33, 63, 64, 65, 96, 97, 127, 128, 129, 7, 512, 200, 33, 5, 9, 17, 30, 511, 256, 257,
                100, 28, 3]


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("seed", [0, 1])
def test_attention_packed_parity(cuda_lib, f16, seed):
    """BGE-base attention (d = 64, 12 heads) on ragged lengths, bf16 and fp16 planes: every request
    of every pack vs the fp64 oracle.  Tolerance: P and ctx rounded to 16 bits (2^-8 relative for
    bf16, 2^-11 for fp16) on values of O(1)."""
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    H, nh = 768, 12
    rng = np.random.default_rng(100 + seed)
    lengths = np.array(PACK_LENGTHS, np.int32)
    if seed:
        rng.shuffle(lengths)
    T = int(lengths.sum())
    x = rng.normal(0, 1.0, (T, 3 * H))
    qkv, qkv64 = fp16_tensor(x) if f16 else bf16_tensor(x)
    ctx = torch.full((T, H), float("nan"), dtype=torch.float16 if f16 else torch.bfloat16, device="cuda")
    binding.op_attention(attn_layout(qkv, H, nh), torch.from_numpy(lengths).cuda(), H, nh, ctx, f16=f16)
    torch.cuda.synchronize()
    got = to_np(ctx)
    starts = inputs.offsets(lengths)
    tol = 4e-3 if f16 else 2e-2
    for i, L in enumerate(lengths):
        sl = slice(starts[i], starts[i + 1])
        ref = oenc.attention(qkv64[sl, :H], qkv64[sl, H:2 * H], qkv64[sl, 2 * H:], nh)
        err = np.abs(got[sl] - ref).max()
        assert err < tol, (i, int(L), err)


@pytest.mark.parametrize("f16", [False, True])
def test_attention_batch_invariant_across_packs(cuda_lib, f16):
    """A request's ctx is bitwise the same alone, at any 32-row segment of a pack and after a long
    request (its keys are the same 32-key chunks in the same order wherever it lands)."""
    from paper_2505_09142_b200 import binding
    H, nh = 768, 12
    rng = np.random.default_rng(7)
    probe = np.array([20, 45, 90, 128], np.int32)   # 1, 2, 3 and 4 segments
    x = rng.normal(0, 1.0, (int(probe.sum()), 3 * H))
    mk = fp16_tensor if f16 else bf16_tensor
    dt = torch.float16 if f16 else torch.bfloat16

    def run(lengths, xx):
        qkv, _ = mk(xx)
        ctx = torch.zeros((int(lengths.sum()), H), dtype=dt, device="cuda")
        binding.op_attention(attn_layout(qkv, H, nh), torch.from_numpy(lengths).cuda(), H, nh, ctx, f16=f16)
        torch.cuda.synchronize()
        return ctx.cpu()

    po = inputs.offsets(probe)
    alone = [run(probe[i:i + 1], x[po[i]:po[i + 1]]) for i in range(len(probe))]
    fill = rng.normal(0, 1.0, (600, 3 * H))
    for prefix in ([], [5], [33], [70], [31, 1], [300], [3, 3, 3]):
        pre = np.array(prefix, np.int32)
        for i in range(len(probe)):
            L = np.concatenate([pre, probe[i:i + 1], np.array([9], np.int32)]).astype(np.int32)
            npre = int(pre.sum())
            xx = np.concatenate([fill[:npre], x[po[i]:po[i + 1]], fill[npre:npre + 9]])
            got = run(L, xx)[npre:npre + int(probe[i])]
            assert torch.equal(got.view(torch.int16), alone[i].view(torch.int16)), (prefix, int(probe[i]))


@pytest.mark.parametrize("f16", [False, True])
def test_attention_lazy_rescale(cuda_lib, f16):
    """Keys whose magnitude grows along the request (x6 from key 64, x12 from key 192), so the block
    maximum of later 64-key blocks exceeds the running maximum by more than 2^8, except in every third
    query row (scaled to near-flat scores): the lazy O rescale runs for part of a warp's rows (warp-uniform TMEM access, alpha = 1
    in the other rows).  Every request vs the fp64 oracle."""
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    H, nh = 768, 12
    rng = np.random.default_rng(11)
    lengths = np.array([100, 300, 512, 65, 200, 129], np.int32)
    T = int(lengths.sum())
    x = rng.normal(0, 1.0, (T, 3 * H))
    starts = inputs.offsets(lengths)
    for i, L in enumerate(lengths):
        pos = np.arange(L)
        scale = np.where(pos >= 192, 12.0, np.where(pos >= 64, 6.0, 1.0))
        x[starts[i]:starts[i + 1], H:2 * H] *= scale[:, None]
        x[starts[i]:starts[i + 1]:3, :H] *= 0.01  # every third query row: flat scores, no rescale
    qkv, qkv64 = fp16_tensor(x) if f16 else bf16_tensor(x)
    ctx = torch.full((T, H), float("nan"), dtype=torch.float16 if f16 else torch.bfloat16, device="cuda")
    binding.op_attention(attn_layout(qkv, H, nh), torch.from_numpy(lengths).cuda(), H, nh, ctx, f16=f16)
    torch.cuda.synchronize()
    got = to_np(ctx)
    tol = 4e-3 if f16 else 2e-2
    for i, L in enumerate(lengths):
        sl = slice(starts[i], starts[i + 1])
        ref = oenc.attention(qkv64[sl, :H], qkv64[sl, H:2 * H], qkv64[sl, 2 * H:], nh)
        err = np.abs(got[sl] - ref).max()
        assert err < tol, (i, int(L), err)


def test_attention_single_token_is_v(cuda_lib):
    """L = 1 closed form on the GPU: ctx = v (up to bf16 of a bf16 value: exact)."""
    from paper_2505_09142_b200 import binding
    H, nh = 768, 12
    lengths = np.ones(5, np.int32)
    rng = np.random.default_rng(3)
    qkv, qkv64 = bf16_tensor(rng.normal(0, 1.0, (5, 3 * H)))
    ctx = torch.empty(5, H, dtype=torch.bfloat16, device="cuda")
    binding.op_attention(attn_layout(qkv, H, nh), torch.from_numpy(lengths).cuda(), H, nh, ctx)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_np(ctx), qkv64[:, 2 * H:])


@pytest.mark.parametrize("H", [128, 768, 1024])
def test_layernorm_parity(cuda_lib, H):
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    rng = np.random.default_rng(H)
    rows = 333
    u = rng.normal(0.5, 3.0, (rows, H)).astype(np.float32)
    g = (1 + rng.uniform(-0.1, 0.1, H)).astype(np.float32)
    b = rng.normal(0, 0.02, H).astype(np.float32)
    out = torch.empty(rows, H, device="cuda")
    outb = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
    binding.op_layernorm(torch.from_numpy(u).cuda(), torch.from_numpy(g).cuda(), torch.from_numpy(b).cuda(),
                         1e-12, out, outb)
    torch.cuda.synchronize()
    ref = oenc.layer_norm(u.astype(np.float64), g, b, 1e-12)
    np.testing.assert_allclose(to_np(out), ref, rtol=0, atol=5e-6)
    np.testing.assert_allclose(to_np(outb), ref, rtol=8e-3, atol=1e-6)


@pytest.mark.parametrize("n,N,K", [(1, 1024, 768), (37, 1024, 1024), (256, 1024, 128), (300, 1000, 1024)])
def test_fc_f32_parity(cuda_lib, n, N, K):
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    rng = np.random.default_rng(n + N + K)
    X = rng.normal(0, 1, (n, K)).astype(np.float32)
    W = (rng.normal(0, 1, (N, K)) * np.sqrt(2.0 / K)).astype(np.float32)
    b = rng.normal(0, 0.1, N).astype(np.float32)
    for relu in (0, 1):
        Y = torch.empty(n, N, device="cuda")
        binding.op_fc_f32(torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), Y,
                          relu)
        torch.cuda.synchronize()
        ref = oenc.linear(X, W, b)
        if relu:
            ref = np.maximum(ref, 0)
        np.testing.assert_allclose(to_np(Y), ref, rtol=2e-5, atol=2e-5)
        # split-K (these shapes take 1-8 splits): the tickets reset, so a repeat is bit-identical
        Y2 = torch.empty(n, N, device="cuda")
        binding.op_fc_f32(torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), Y2,
                          relu)
        torch.cuda.synchronize()
        assert torch.equal(Y, Y2)


@pytest.mark.parametrize("M,N,K", [(300, 768, 768), (1000, 768, 3072), (129, 1024, 1024), (129, 1024, 4096),
                                   (77, 128, 128), (200, 128, 512), (1, 768, 768), (5000, 768, 768)])
def test_gemm_fused_residual_layernorm_parity(cuda_lib, M, N, K):
    """Attention-output / FFN2 GEMM with the cluster-fused residual + LayerNorm epilogue
    (row statistics exchanged over DSMEM) vs oracle linear -> + residual -> layer_norm."""
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    rng = np.random.default_rng(M + N + K)
    A, A64 = bf16_tensor(rng.normal(0, 1, (M, K)))
    W, W64 = bf16_tensor(rng.normal(0, 0.03, (N, K)))
    b = rng.normal(0, 0.1, N).astype(np.float32)
    res = rng.normal(0.2, 1.5, (M, N)).astype(np.float32)
    g = (1 + rng.uniform(-0.1, 0.1, N)).astype(np.float32)
    be = rng.normal(0, 0.02, N).astype(np.float32)
    h = torch.from_numpy(res.copy()).cuda()
    hb = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    binding.op_gemm_ln(A, W, torch.from_numpy(b).cuda(), h, torch.from_numpy(g).cuda(), torch.from_numpy(be).cuda(),
                       1e-12, hb)
    torch.cuda.synchronize()
    ref = oenc.layer_norm(oenc.linear(A64, W64, b) + res, g, be, 1e-12)
    np.testing.assert_allclose(to_np(h), ref, rtol=0, atol=2e-4)
    np.testing.assert_allclose(to_np(hb), ref, rtol=8e-3, atol=1e-5)


@pytest.mark.parametrize("M,N,K", [(300, 768, 768), (1000, 768, 3072), (129, 1024, 1024), (77, 256, 128),
                                   (1, 768, 768), (5000, 768, 768)])
def test_gemm_fused_residual16_layernorm_parity(cuda_lib, M, N, K):
    """The fp16-residual LayerNorm epilogue (EPI_BIAS_RESID16_LN, elis_config.residual16):
    fp16 A / W / residual, fp32 v and statistics, fp16 LN output written in place over the
    residual -- vs the oracle on the same fp16-representable inputs, to one fp16 rounding."""
    from paper_2505_09142_b200 import binding
    from oracle import encoder as oenc
    rng = np.random.default_rng(M + N + K + 1)
    A = torch.from_numpy(rng.normal(0, 1, (M, K))).half()
    W = torch.from_numpy(rng.normal(0, 0.03, (N, K))).half()
    res = torch.from_numpy(rng.normal(0.2, 1.5, (M, N))).half()
    b = rng.normal(0, 0.1, N).astype(np.float32)
    g = (1 + rng.uniform(-0.1, 0.1, N)).astype(np.float32)
    be = rng.normal(0, 0.02, N).astype(np.float32)
    h = res.cuda()
    binding.op_gemm_ln16(A.cuda(), W.cuda(), torch.from_numpy(b).cuda(), h, torch.from_numpy(g).cuda(),
                         torch.from_numpy(be).cuda(), 1e-12)
    torch.cuda.synchronize()
    ref = oenc.layer_norm(oenc.linear(A.double().numpy(), W.double().numpy(), b) + res.double().numpy(), g, be, 1e-12)
    got = h.float().cpu().numpy().astype(np.float64)
    # one fp16 rounding of |y| <= ~6 (2^-9 relative) plus the fp32 accumulation
    np.testing.assert_allclose(got, ref, rtol=1.5e-3, atol=2e-4)


@pytest.mark.parametrize("M", [1000, 43296, 77])
def test_gemm_ln16_global_stats_bitwise_equal_cluster(cuda_lib, M):
    """FFN2's LayerNorm statistics through global memory (CTA pairs without a shared cluster, the
    grid on every SM) give bit-identical rows to the cluster / DSMEM exchange: the partials are
    merged in the same n order."""
    from paper_2505_09142_b200 import binding
    rng = np.random.default_rng(M)
    K, N = 3072, 768
    A = torch.from_numpy(rng.normal(0, 1, (M, K))).half().cuda()
    W = torch.from_numpy(rng.normal(0, 0.02, (N, K))).half().cuda()
    res = torch.from_numpy(rng.normal(0.2, 1.5, (M, N))).half().cuda()
    b = torch.from_numpy(rng.normal(0, 0.1, N).astype(np.float32)).cuda()
    g = torch.from_numpy((1 + rng.uniform(-0.1, 0.1, N)).astype(np.float32)).cuda()
    be = torch.from_numpy(rng.normal(0, 0.02, N).astype(np.float32)).cuda()
    h_cl, h_gx = res.clone(), res.clone()
    binding.op_gemm_ln16(A, W, b, h_cl, g, be, 1e-12, global_stats=False)
    binding.op_gemm_ln16(A, W, b, h_gx, g, be, 1e-12, global_stats=True)
    torch.cuda.synchronize()
    assert torch.equal(h_cl, h_gx)
    assert torch.isfinite(h_gx.float()).all()

"""K1-K5 kernel parity on the B200 against the numpy oracle (oracle/ops.py).

Bars: dropout keep-masks bit-exact (Philox integer compare); pack and the
offload->reload round trip bit-exact; LayerNorm / GeLU within bf16 output
rounding (stated per test)."""

import numpy as np
import pytest

from oracle import ops as ref
from oracle.philox import keep_mask

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2503_01328_b200.runtime import native  # noqa: E402

DEV = torch.device("cuda:0")


def bf(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(DEV).bfloat16()


def npf(t):
    return t.float().cpu().numpy()


@pytest.mark.parametrize("n,p,seed,offset", [(8, 0.1, 42, 0), (4096, 0.1, 42, 7), (1 << 20, 0.5, 2**40 + 3, 2**33 + 5), (64, 0.0, 1, 1)])
def test_dropout_mask_bit_exact(n, p, seed, offset):
    x = torch.ones(n, device=DEV, dtype=torch.bfloat16)
    y = torch.empty_like(x)
    native.dropout(x, y, p, seed, offset)
    torch.cuda.synchronize()
    got = npf(y) != 0
    assert np.array_equal(got, keep_mask(n, p, seed, offset))
    if p > 0:
        kept = npf(y)[got]
        assert np.all(kept == np.float32(ref.bf16_round(np.float32(1.0 / (1.0 - p)))))


@pytest.mark.parametrize("rows,h", [(1, 256), (37, 256), (512, 2048), (64, 5120), (16, 8192), (9, 264)])
def test_layernorm_fwd(rows, h):
    rng = np.random.default_rng(rows * h)
    x = ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32) * 3 + 1)
    gamma = rng.standard_normal(h).astype(np.float32)
    beta = rng.standard_normal(h).astype(np.float32)
    y = torch.empty(rows, h, device=DEV, dtype=torch.bfloat16)
    native.layernorm_fwd(bf(x), torch.from_numpy(gamma).to(DEV), torch.from_numpy(beta).to(DEV), y)
    want = ref.layernorm(x, gamma, beta)
    # bf16 output: |err| <= 2^-8 relative of the value (+ tiny fp32 reduction slack)
    np.testing.assert_allclose(npf(y), want, rtol=2 ** -8, atol=1e-3 * np.abs(gamma).max())


@pytest.mark.parametrize("rows,h,p", [(300, 256, 0.1), (128, 2048, 0.1), (33, 4096, 0.0), (45, 5120, 0.1), (20, 8192, 0.1)])
def test_residual_dropout_ln(rows, h, p):
    rng = np.random.default_rng(h)
    resid = ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32))
    branch = ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32))
    gamma = (1 + 0.1 * rng.standard_normal(h)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(h)).astype(np.float32)
    out = torch.empty(rows, h, device=DEV, dtype=torch.bfloat16)
    ln = torch.empty_like(out)
    native.residual_dropout_ln_fwd(bf(resid), bf(branch), out, torch.from_numpy(gamma).to(DEV),
                                   torch.from_numpy(beta).to(DEV), ln, p, 42, 99)
    want_out = ref.residual_dropout(resid, branch, p, 42, 99)
    # out = bf16(resid + mask*branch*scale): the device may fuse the multiply-add
    # (one rounding instead of two) -> at most 1 bf16 ulp apart, masks identical
    assert ref.bf16_ulp_diff(npf(out), want_out).max() <= 1
    np.testing.assert_allclose(npf(ln), ref.layernorm(npf(out), gamma, beta), rtol=2 ** -7, atol=2e-2)


@pytest.mark.parametrize("rows,h,with_resid,p", [(200, 256, True, 0.1), (64, 2048, False, 0.0), (40, 5120, True, 0.1),
                                                 (70, 1536, True, 0.0), (300, 4096, True, 0.1), (30, 6144, False, 0.1),
                                                 (50, 8192, True, 0.1)])
def test_layernorm_bwd(rows, h, with_resid, p):
    rng = np.random.default_rng(rows + h)
    x = ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32) * 2)
    dy = ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32))
    rg = ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32))
    gamma = (1 + 0.1 * rng.standard_normal(h)).astype(np.float32)
    dx = torch.empty(rows, h, device=DEV, dtype=torch.bfloat16)
    drop = torch.empty_like(dx) if p > 0 else None
    dgamma = torch.zeros(h, device=DEV)
    dbeta = torch.zeros(h, device=DEV)
    native.layernorm_bwd(bf(x), torch.from_numpy(gamma).to(DEV), bf(dy), bf(rg) if with_resid else None, dx, dgamma,
                         dbeta, drop_out=drop, p=p, drop_seed=5, drop_offset=11)
    want_dx, want_dg, want_db = ref.layernorm_bwd(x, gamma, dy)
    if with_resid:
        want_dx = want_dx + rg
    np.testing.assert_allclose(npf(dx), want_dx, rtol=2 ** -7, atol=3e-2)
    np.testing.assert_allclose(dgamma.cpu().numpy(), want_dg, rtol=1e-3, atol=1e-3 * rows)
    np.testing.assert_allclose(dbeta.cpu().numpy(), want_db, rtol=1e-3, atol=1e-3 * rows)
    if drop is not None:
        # bit-exact: the fused replay equals the standalone dropout of the stored dx
        alone = torch.empty_like(dx)
        native.dropout(dx, alone, p, 5, 11)
        assert torch.equal(alone, drop)


@pytest.mark.parametrize("rows,h", [(200, 256), (64, 2048), (40, 5120), (30, 8192)])
def test_layernorm_bwd_emits_ln_recompute(rows, h):
    """ln_out: the LN recompute emitted by the backward equals LN(x) (oracle, bf16
    rounding) and is 1 ulp-close to the standalone forward; dx is unchanged by it."""
    rng = np.random.default_rng(3 * rows + h)
    x = ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32) * 2)
    dy = ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32))
    gamma = (1 + 0.1 * rng.standard_normal(h)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(h)).astype(np.float32)
    g_, b_ = torch.from_numpy(gamma).to(DEV), torch.from_numpy(beta).to(DEV)
    outs = []
    for with_ln in (False, True):
        dx = torch.empty(rows, h, device=DEV, dtype=torch.bfloat16)
        ln = torch.empty_like(dx) if with_ln else None
        dgamma, dbeta = torch.zeros(h, device=DEV), torch.zeros(h, device=DEV)
        native.layernorm_bwd(bf(x), g_, bf(dy), None, dx, dgamma, dbeta, beta=b_ if with_ln else None, ln_out=ln)
        outs.append((dx, ln))
    assert torch.equal(outs[0][0], outs[1][0])
    ln = outs[1][1]
    np.testing.assert_allclose(npf(ln), ref.layernorm(x, gamma, beta), rtol=2 ** -7, atol=2e-2)
    alone = torch.empty_like(ln)
    native.layernorm_fwd(bf(x), g_, b_, alone)
    assert ref.bf16_ulp_diff(npf(ln), npf(alone)).max() <= 1
    with pytest.raises(native.PpoError):  # ln_out needs beta
        native.layernorm_bwd(bf(x), g_, bf(dy), None, outs[0][0], dgamma, dbeta, ln_out=ln)


@pytest.mark.parametrize("rows,h", [(100, 256), (64, 2048), (33, 4096), (20, 5120), (12, 8192)])
def test_layernorm_fwd2(rows, h):
    """Two LayerNorms in one launch == two standalone launches, bit for bit."""
    rng = np.random.default_rng(rows * 7 + h)
    x, h1 = (ref.bf16_round(rng.standard_normal((rows, h)).astype(np.float32) * 2) for _ in range(2))
    p = [torch.from_numpy((1 + 0.1 * rng.standard_normal(h)).astype(np.float32)).to(DEV) for _ in range(2)]
    q = [torch.from_numpy((0.1 * rng.standard_normal(h)).astype(np.float32)).to(DEV) for _ in range(2)]
    ln1, ln2 = (torch.empty(rows, h, device=DEV, dtype=torch.bfloat16) for _ in range(2))
    native.layernorm_fwd2(bf(x), p[0], q[0], ln1, bf(h1), p[1], q[1], ln2)
    for got, src, gm, bt in ((ln1, x, p[0], q[0]), (ln2, h1, p[1], q[1])):
        alone = torch.empty_like(got)
        native.layernorm_fwd(bf(src), gm, bt, alone)
        assert torch.equal(got, alone)


@pytest.mark.parametrize("n", [8, 4096, 1 << 20])
def test_gelu_fwd_bwd(n):
    rng = np.random.default_rng(n)
    f = ref.bf16_round(rng.standard_normal(n).astype(np.float32) * 3)
    dg = ref.bf16_round(rng.standard_normal(n).astype(np.float32))
    g = torch.empty(n, device=DEV, dtype=torch.bfloat16)
    native.gelu_fwd(bf(f), g)
    np.testing.assert_allclose(npf(g), ref.gelu(f), rtol=2 ** -7, atol=1e-6)
    g2 = torch.empty_like(g)
    df = bf(dg)
    native.gelu_bwd(bf(f), df, g2, df)  # df aliases dg (in place)
    assert torch.equal(g, g2)
    # tanh.approx.f32 (SFU) has ~2^-11 absolute error: atol covers it where gelu' ~ 0
    np.testing.assert_allclose(npf(df), dg * ref.gelu_grad(f), rtol=2 ** -7, atol=1e-3)


def test_pack_gather_bit_exact():
    rng = np.random.default_rng(3)
    a = rng.integers(0, 256, 4096 * 3, dtype=np.uint8)
    b = rng.integers(0, 256, 64 * 96, dtype=np.uint8)  # 64 rows x 96 B, pitch 96, take 48 B/row
    ta, tb = torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV)
    dst = torch.zeros(16384, dtype=torch.uint8, device=DEV)
    items = [(ta, 0, 1, a.size, 0), (tb, 12288, 64, 48, 96)]
    native.pack(items, dst)
    want = ref.pack([(a, 0, 1, a.size, 0), (b, 12288, 64, 48, 96)], 16384)
    assert np.array_equal(dst.cpu().numpy(), want)


@pytest.mark.parametrize("sizes", [(16 * 1024 * 1024 + 48, 262144, 16), (1 << 20,), (3 * 16384 + 32, 5 << 20)])
def test_pack_tma_bulk_bit_exact(sizes):
    """Contiguous items >= 1 MiB in total take the TMA bulk path (cp.async.bulk
    global->smem->global, 16 KiB chunks, ragged tails); every byte lands exactly
    where the numpy restatement puts it, and nothing outside the items is touched."""
    rng = np.random.default_rng(len(sizes))
    srcs = [rng.integers(0, 256, n, dtype=np.uint8) for n in sizes]
    offs, acc = [], 32
    for n in sizes:
        offs.append(acc)
        acc += (n + 255) // 256 * 256 + 64
    total = acc + 128
    dst = torch.full((total,), 0xA5, dtype=torch.uint8, device=DEV)
    items = [(torch.from_numpy(x).to(DEV), o, 1, x.size, 0) for x, o in zip(srcs, offs)]
    native.pack(items, dst)
    want = np.full(total, 0xA5, dtype=np.uint8)
    want = ref.pack([(x, o, 1, x.size, 0) for x, o in zip(srcs, offs)], total, base=want)
    assert np.array_equal(dst.cpu().numpy(), want)


def test_offload_reload_round_trip_bit_exact():
    """K2: device slab -> pinned bins -> fresh device slab, every byte identical."""
    from paper_2503_01328_b200.runtime.layout import make_layout

    lay = make_layout(layers=2, seq=512, hidden=256, heads=4, head_grad=True)
    src = torch.randint(0, 256, (lay.slab_bytes,), dtype=torch.uint8, device=DEV)
    back = torch.zeros_like(src)
    pool = native.PinnedPool(lay.host_bytes + 8192)
    bins = tuple(pool.carve(b) for b in lay.bins)
    copy = torch.cuda.Stream()
    done_out, done_in = torch.cuda.Event(), torch.cuda.Event()
    ready = torch.cuda.Event()
    ready.record()
    native.transfer(native.PPO_D2H, lay.segments(src.data_ptr(), bins), copy.cuda_stream, ready.cuda_event, None)
    done_out.record(copy)
    native.transfer(native.PPO_H2D, lay.segments(back.data_ptr(), bins), copy.cuda_stream, None, None)
    done_in.record(copy)
    done_in.synchronize()
    assert torch.equal(src, back)
    assert lay.payload_bytes == 2 * 20 * 512 * 256
    pool.close()


@pytest.mark.parametrize("M,N,K", [(512, 768, 256), (4096, 2048, 2048), (256, 1024, 512)])
def test_tcgen05_gemms_match_fp32(M, N, K):
    """K6: the tcgen05 GEMMs (TN fwd, NN dgrad, fp32-accumulating wgrad, fused GeLU /
    dGeLU epilogues) against fp32 references; bf16 outputs -> rel. L2 < 5e-3 (1e-2 with
    the SFU tanh of the fused activations)."""
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    a = (torch.randn(M, K, generator=g) * 0.5).to(DEV).bfloat16()
    w = (torch.randn(N, K, generator=g) * 0.05).to(DEV).bfloat16()

    def rel(x, y):
        return float((x.float() - y).norm() / y.norm())

    d = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    native.gemm_tn(a, w, d)
    want = a.float() @ w.float().t()
    assert rel(d, want) < 5e-3
    f, gg = torch.empty_like(d), torch.empty_like(d)
    native.gemm_tn_gelu(a, w, gg, f, torch.zeros(N, device=DEV))
    assert rel(f, want) < 5e-3
    assert rel(gg, torch.from_numpy(ref.gelu(want.cpu().numpy())).to(DEV)) < 1e-2
    # NN: d2[M,K] = d[M,N] @ w[N,K]
    d2 = torch.empty(M, K, device=DEV, dtype=torch.bfloat16)
    native.gemm_nn(d, w, d2)
    d3 = d2.clone()
    native.gemm_nn(d, w, d3, 1.0)
    assert rel(d3, 2 * (d.float() @ w.float())) < 5e-3
    assert rel(d2, d.float() @ w.float()) < 5e-3
    # fused dGeLU: (d @ w) * gelu'(z)
    z = torch.randn(M, K, generator=g).to(DEV).bfloat16()
    native.gemm_nn_dgelu(d, w, z, d2)
    dz = torch.from_numpy(ref.gelu_grad(z.float().cpu().numpy())).to(DEV)
    assert rel(d2, (d.float() @ w.float()) * dz) < 1e-2
    # wgrad: acc[N,K] += d[M,N]^T @ a[M,K] (fp32 accumulation, beta = 1)
    acc = torch.randn(N, K, device=DEV)
    want = acc + d.float().t() @ a.float()
    native.gemm_wgrad(d, a, acc, 1.0)
    assert rel(acc, want) < 1e-4


@pytest.mark.parametrize("rows,h,vocab", [(512, 256, 1024), (4096, 2048, 50304), (8, 8, 3)])
def test_embedding_fwd_bwd(rows, h, vocab):
    """First-stage embedding: forward bit-exact vs torch (one bf16 rounding of the
    sum); backward = fp32 index_add of the bf16 gradient (atomics: order-free up to
    fp32 rounding), with repeated tokens."""
    g = torch.Generator(device="cpu").manual_seed(rows + h)
    tok = torch.randint(0, vocab, (rows,), generator=g)
    tok[: rows // 4] = tok[0]  # many repeats of one token
    tok = tok.to(DEV)
    wte = (torch.randn(vocab, h, generator=g) * 0.02).to(DEV, torch.bfloat16)
    wpe = (torch.randn(rows, h, generator=g) * 0.02).to(DEV, torch.bfloat16)
    x = torch.empty(rows, h, device=DEV, dtype=torch.bfloat16)
    native.embed_fwd(tok, wte, wpe, x)
    want = torch.nn.functional.embedding(tok, wte) + wpe
    assert torch.equal(x, want)
    dy = (torch.randn(rows, h, generator=g)).to(DEV, torch.bfloat16)
    gwte = torch.randn(vocab, h, device=DEV)
    gwpe = torch.randn(rows, h, device=DEV)
    w_te, w_pe = gwte.clone().index_add_(0, tok, dy.float()), gwpe + dy.float()
    native.embed_bwd(tok, dy, gwte, gwpe)
    torch.cuda.synchronize()
    assert torch.equal(gwpe, w_pe)
    torch.testing.assert_close(gwte, w_te, rtol=1e-5, atol=1e-4 * max(1.0, rows / 64))


@pytest.mark.parametrize("nbytes", [16, 4096 * 2048 * 2 + 6])
def test_nccl_p2p_self_loop(nbytes):
    """K8 on hardware with one GPU: a 1-rank NCCL communicator sends to and receives
    from itself in one grouped ppo_p2p call (the same ncclGroupStart/ncclSend/ncclRecv
    path the pipeline's 2-rank edge communicators use); bytes arrive bit-exact."""
    comm = native.NcclComm(native.NcclComm.unique_id(), 1, 0, 0)
    try:
        src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=DEV)
        dst = torch.zeros_like(src)
        stream = torch.cuda.Stream(DEV)
        stream.wait_stream(torch.cuda.current_stream(DEV))
        comm.p2p([(True, 0, src.data_ptr(), nbytes), (False, 0, dst.data_ptr(), nbytes)], stream.cuda_stream)
        stream.synchronize()
        assert torch.equal(src, dst)
        with pytest.raises(native.PpoError):
            comm.p2p([(True, 1, src.data_ptr(), nbytes)], stream.cuda_stream)  # peer out of range
    finally:
        comm.close()


def test_gemm_swizzle_bit_identical_and_tuner(tmp_path):
    """The tile-scheduler swizzle only reorders whole output tiles: results are
    bit-identical across swizzles; the gemm="auto" tuner records a measured choice."""
    from paper_2503_01328_b200.runtime import gemm_tune
    from paper_2503_01328_b200.runtime.model import ModelConfig, Stage

    M, N, K = 1024, 1536, 512
    a = (torch.randn(M, K, device=DEV) * 0.5).bfloat16()
    b = (torch.randn(N, K, device=DEV) * 0.5).bfloat16()
    outs = []
    for sw in (1, 2, 8):
        native.gemm_set_swizzle("tn", M, N, K, sw)
        d = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
        native.gemm_tn(a, b, d)
        outs.append(d)
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    ref = a.float() @ b.float().t()
    assert float((outs[0].float() - ref).norm() / ref.norm()) < 1e-2
    with pytest.raises(native.PpoError):
        native.gemm_set_swizzle("tn", M, N, K, 3)  # not a power of two
    st = Stage(ModelConfig(n_layers=1, hidden=256, heads=4, seq=512, vocab=512), 0, 1, 1, DEV, gemm="auto")
    x = (torch.randn(512, 256, device=DEV) * 0.5).bfloat16()
    w = (torch.randn(768, 256, device=DEV) * 0.5).bfloat16()
    y = torch.empty(512, 768, device=DEV, dtype=torch.bfloat16)
    st.mm_fwd(x, w, y)
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t()
    assert float((y.float() - ref).norm() / ref.norm()) < 1e-2
    dec = gemm_tune.decisions()
    assert "tn 512x768x256" in dec and dec["tn 512x768x256"]["backend"] in ("tcgen05", "cublas")
    assert dec["tn 512x768x256"]["swizzle"] in gemm_tune.SWIZZLES
    # every layer shape was decided at Stage construction: pass bodies only look up
    assert not gemm_tune.MISSES
    assert all(gemm_tune.gemm_key(k, sh) in dec for (k, *sh) in gemm_tune.layer_gemm_shapes(512, 256))
    # a saved table reloads to the same decisions (same digest)
    d0 = gemm_tune.digest()
    path = str(tmp_path / "table.json")
    gemm_tune.save(path)
    gemm_tune.reset()
    gemm_tune.load(path)
    assert gemm_tune.digest() == d0


def _attn_ref(qkv: torch.Tensor, heads: int):
    """fp32 causal attention on the device: o [s, h] and natural-log lse [heads, s]."""
    s, h3 = qkv.shape
    h = h3 // 3
    D = h // heads
    q, k, v = qkv.float().view(s, 3, heads, D).permute(1, 2, 0, 3)  # [heads, s, D] each
    scores = (q @ k.transpose(1, 2)) * D ** -0.5
    mask = torch.ones(s, s, device=qkv.device, dtype=torch.bool).triu(1)
    scores = scores.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(scores, dim=-1)  # [heads, s]
    o = torch.softmax(scores, dim=-1) @ v  # [heads, s, D]
    return o.transpose(0, 1).reshape(s, h), lse


@pytest.mark.parametrize("s,heads,D", [(256, 4, 64), (512, 4, 64), (1024, 8, 128), (2048, 2, 128)])
def test_attn_fwd_matches_fp32(s, heads, D):
    """K7 (tcgen05 causal attention forward) against fp32 attention on the same bf16
    inputs: o within bf16 rounding of P (rel. L2 <= 1e-2, max abs <= 2e-2 at unit-scale
    inputs), lse within 2e-3 absolute (fp32 statistics, exp2-based softmax)."""
    g = torch.Generator(device=DEV).manual_seed(s + heads + D)
    qkv = torch.randn(s, 3 * heads * D, device=DEV, generator=g).bfloat16()
    o = torch.full((s, heads * D), float("nan"), device=DEV, dtype=torch.bfloat16)
    lse = torch.full((heads, s), float("nan"), device=DEV, dtype=torch.float32)
    native.attn_fwd(qkv, o, lse, heads)
    torch.cuda.synchronize()
    o_ref, lse_ref = _attn_ref(qkv, heads)
    assert torch.isfinite(o.float()).all() and torch.isfinite(lse).all()
    rel = ((o.float() - o_ref).norm() / o_ref.norm()).item()
    assert rel <= 1e-2, rel
    assert (o.float() - o_ref).abs().max().item() <= 2e-2
    assert (lse - lse_ref).abs().max().item() <= 2e-3


def test_attn_fwd_matches_cudnn_at_c2_shape():
    """At the C2 attention shape (s=4096, 16 heads of 128) our o and lse match cuDNN's
    fused forward -- the statistics feed cuDNN's backward, so they must be the same
    quantity (natural-log logsumexp, [heads, s])."""
    s, heads, D = 4096, 16, 128
    g = torch.Generator(device=DEV).manual_seed(7)
    qkv = torch.randn(s, 3 * heads * D, device=DEV, generator=g).bfloat16()
    o = torch.empty(s, heads * D, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(heads, s, device=DEV, dtype=torch.float32)
    native.attn_fwd(qkv, o, lse, heads)
    q, k, v = [t.transpose(1, 2) for t in qkv.view(1, s, 3, heads, D).unbind(2)]
    res = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
    torch.cuda.synchronize()
    o_cud = res[0].transpose(1, 2).reshape(s, heads * D).float()
    lse_cud = res[1].reshape(heads, s)
    assert (lse - lse_cud).abs().max().item() <= 2e-3
    rel = ((o.float() - o_cud).norm() / o_cud.norm()).item()
    assert rel <= 1e-2, rel


def test_attn_fwd_rejects_bad_shapes():
    qkv = torch.zeros(300, 3 * 256, device=DEV, dtype=torch.bfloat16)  # seq not a multiple of 256
    with pytest.raises(native.PpoError):
        native.attn_fwd(qkv, torch.empty(300, 256, device=DEV, dtype=torch.bfloat16),
                        torch.empty(4 * 300, device=DEV), 4)
    qkv = torch.zeros(256, 3 * 96 * 2, device=DEV, dtype=torch.bfloat16)  # head_dim 96
    with pytest.raises(native.PpoError):
        native.attn_fwd(qkv, torch.empty(256, 192, device=DEV, dtype=torch.bfloat16),
                        torch.empty(2 * 256, device=DEV), 2)

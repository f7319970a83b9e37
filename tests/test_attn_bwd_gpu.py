"""K7b (hand-written tcgen05 causal attention backward) against an fp32 reference of the
same op on the same bf16 inputs, and against cuDNN's fused backward at the C2 shape.

Bars: dq, dk, dv each within 1e-2 relative L2 of fp32 autograd (the kernel rounds P and
dS to bf16 for the tensor core, as every flash backward does; observed ~3-5e-3), and no
non-finite values.  The reference prices this op only through its FLOP model
(pkg/src/ppoff/costs.py:144-161)."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2503_01328_b200.runtime import native  # noqa: E402

DEV = torch.device("cuda:0")


def _fp32_grads(qkv, do, heads):
    """fp32 causal attention backward by autograd: o [s, h], lse [heads, s], dqkv [s, 3h]."""
    s, h3 = qkv.shape
    h = h3 // 3
    D = h // heads
    x = qkv.float().clone().requires_grad_(True)
    q, k, v = x.view(s, 3, heads, D).permute(1, 2, 0, 3)
    scores = (q @ k.transpose(1, 2)) * D ** -0.5
    mask = torch.ones(s, s, device=qkv.device, dtype=torch.bool).triu(1)
    scores = scores.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(scores, dim=-1)
    o = (torch.softmax(scores, dim=-1) @ v).transpose(0, 1).reshape(s, h)
    o.backward(do.float())
    return o.detach(), lse.detach(), x.grad


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def _run_ours(qkv, o, do, lse, heads):
    s, h3 = qkv.shape
    dqkv = torch.full_like(qkv, float("nan"))
    ws = torch.empty(native.attn_bwd_workspace_bytes(s, heads, h3 // 3 // heads), device=DEV, dtype=torch.uint8)
    native.attn_bwd(qkv, o, do, lse, dqkv, heads, ws)
    torch.cuda.synchronize()
    return dqkv


@pytest.mark.parametrize("s,heads,D", [(128, 1, 128), (256, 2, 128), (512, 4, 128), (1024, 2, 128), (2048, 3, 128),
                                       (128, 2, 64), (256, 4, 64), (512, 4, 64), (1024, 3, 64)])
def test_attn_bwd_matches_fp32(s, heads, D):
    h = heads * D
    g = torch.Generator(device=DEV).manual_seed(11 * s + heads)
    qkv = torch.randn(s, 3 * h, device=DEV, generator=g).bfloat16()
    do = torch.randn(s, h, device=DEV, generator=g).bfloat16()
    o_ref, lse_ref, dqkv_ref = _fp32_grads(qkv, do, heads)
    # the saved set as the forward leaves it: o in bf16, lse in fp32 (our forward kernel)
    o = torch.empty(s, h, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(heads, s, device=DEV, dtype=torch.float32)
    if s % 256 == 0:
        native.attn_fwd(qkv, o, lse, heads)
    else:
        o.copy_(o_ref)
        lse.copy_(lse_ref)
    dqkv = _run_ours(qkv, o, do, lse, heads)
    assert torch.isfinite(dqkv.float()).all()
    for j, name in enumerate(("dq", "dk", "dv")):
        got, want = dqkv[:, j * h:(j + 1) * h], dqkv_ref[:, j * h:(j + 1) * h]
        assert _rel(got, want) <= 1e-2, (name, _rel(got, want))


def test_attn_bwd_matches_cudnn_at_c2_shape():
    """C2 (s=4096, 16 heads of 128): our backward against cuDNN's fused backward fed the
    same saved o and lse."""
    s, heads, D = 4096, 16, 128
    h = heads * D
    g = torch.Generator(device=DEV).manual_seed(5)
    qkv = torch.randn(s, 3 * h, device=DEV, generator=g).bfloat16()
    do = torch.randn(s, h, device=DEV, generator=g).bfloat16()
    q, k, v = [t.transpose(1, 2) for t in qkv.view(1, s, 3, heads, D).unbind(2)]
    res = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
    o4, lse4 = res[0], res[1]
    do4 = do.view(1, s, heads, D).transpose(1, 2)
    dq, dk, dv = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
        do4, q, k, v, o4, lse4, res[6], res[7], None, res[2], res[3], res[4], res[5], 0.0, True)
    o = o4.transpose(1, 2).reshape(s, h).contiguous()
    lse = lse4.reshape(heads, s).contiguous()
    dqkv = _run_ours(qkv, o, do, lse, heads)
    for j, ref in enumerate((dq, dk, dv)):
        want = ref.transpose(1, 2).reshape(s, h)
        got = dqkv[:, j * h:(j + 1) * h]
        assert _rel(got, want) <= 1e-2, (j, _rel(got, want))


def test_attn_bwd_rejects_bad_shapes():
    heads = 2
    qkv = torch.zeros(200, 3 * 256, device=DEV, dtype=torch.bfloat16)  # seq not a multiple of 128
    o = torch.zeros(200, 256, device=DEV, dtype=torch.bfloat16)
    ws = torch.empty(native.attn_bwd_workspace_bytes(256, heads, 128), device=DEV, dtype=torch.uint8)
    with pytest.raises(native.PpoError):
        native.attn_bwd(qkv, o, o, torch.zeros(heads, 200, device=DEV), torch.empty_like(qkv), heads, ws)
    qkv = torch.zeros(256, 3 * 192, device=DEV, dtype=torch.bfloat16)  # head_dim 96
    o = torch.zeros(256, 192, device=DEV, dtype=torch.bfloat16)
    with pytest.raises(native.PpoError):
        native.attn_bwd(qkv, o, o, torch.zeros(heads, 256, device=DEV), torch.empty_like(qkv), heads, ws)


@pytest.mark.parametrize("s,heads,D", [(8192, 16, 128), (8192, 32, 64), (16384, 40, 128)])
def test_attention_matches_cudnn_grouped_persistent(s, heads, D):
    """Shapes where both kernels dispatch in head groups (forward: 4sh bytes > 64 MB;
    backward: groups whose Q, dO and fp32 dQ fit ~0.7 of L2 -- 5 of 40 heads at the C4
    shape, the last case) and every persistent CTA walks several items.  Forward o / lse and backward dq / dk / dv against
    cuDNN's fused kernels on the same inputs (o / lse of the forward under test fed to both
    backwards)."""
    h = heads * D
    g = torch.Generator(device=DEV).manual_seed(s + heads)
    qkv = torch.randn(s, 3 * h, device=DEV, generator=g).bfloat16()
    do = torch.randn(s, h, device=DEV, generator=g).bfloat16()
    o = torch.empty(s, h, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(heads, s, device=DEV, dtype=torch.float32)
    native.attn_fwd(qkv, o, lse, heads)
    q, k, v = [t.transpose(1, 2) for t in qkv.view(1, s, 3, heads, D).unbind(2)]
    res = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
    torch.cuda.synchronize()
    assert _rel(o, res[0].transpose(1, 2).reshape(s, h)) <= 1e-2
    assert (lse - res[1].reshape(heads, s)).abs().max().item() <= 2e-3
    o4 = o.view(1, s, heads, D).transpose(1, 2)
    do4 = do.view(1, s, heads, D).transpose(1, 2)
    dq, dk, dv = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
        do4, q, k, v, o4, lse.view(1, heads, s, 1), res[6], res[7], None, res[2], res[3], res[4], res[5], 0.0, True)
    dqkv = _run_ours(qkv, o, do, lse, heads)
    for j, ref in enumerate((dq, dk, dv)):
        got = dqkv[:, j * h:(j + 1) * h]
        assert _rel(got, ref.transpose(1, 2).reshape(s, h)) <= 1e-2, (j, _rel(got, ref.transpose(1, 2).reshape(s, h)))

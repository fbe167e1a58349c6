"""Kernel-level GPU tests: swap gather/scatter (both engines, Llama3-8B
block shape, ragged token ranges, layer sub-ranges), KV append, paged decode
attention vs an fp32 reference (GQA 32/8 hd128, 4/2 hd64, 40/8), empty and
maximum-size cases."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2510_02758_b200 import _lib

    return _lib


def _pool(cuda, nb, nh, L, H, D):
    from paper_2510_02758_b200.dataplane import KvPool

    p = KvPool(nb, nh, L, H, D, device=cuda)
    g = torch.Generator(device="cpu").manual_seed(0)
    p.gpu.copy_(torch.randint(-32768, 32767, p.gpu.shape, dtype=torch.int16, generator=g).to(cuda))
    p.host.copy_(torch.randint(-32768, 32767, p.host.shape, dtype=torch.int16, generator=g))
    return p


def _segs(lib, segs):
    arr = (lib.TfSeg * max(1, len(segs)))()
    for i, s in enumerate(segs):
        arr[i].gpu_block, arr[i].host_block, arr[i].slot_begin, arr[i].n_slots = s
    return arr


@pytest.mark.parametrize("engine", [0, 1, 2, 3])
@pytest.mark.parametrize("shape", [(2, 2, 64), (32, 8, 128)])
def test_swap_roundtrip(cuda, engine, shape):
    L, H, D = shape
    lib = _lib()
    nb, nh = 48, 40
    p = _pool(cuda, nb, nh, L, H, D)
    rng = np.random.default_rng(engine * 7 + L)
    segs = []
    gb = rng.permutation(nb)[:30]
    hb = rng.permutation(nh)[:30]
    for i in range(30):
        s0 = int(rng.integers(0, 16))
        n = int(rng.integers(1, 17 - s0)) if i % 3 else 16 - (s0 := 0)
        segs.append((int(gb[i]), int(hb[i]), s0, n))
    for l0, l1 in ((0, L), (L // 2, L), (0, 1)):
        before_gpu = p.gpu_view().cpu().clone()
        before_host = p.host_view().clone()
        st = torch.cuda.Stream()
        lib.check(lib.lib.tf_kv_gather_d2h(p.handle, _segs(lib, segs), len(segs), l0, l1, engine,
                                           C.c_void_p(st.cuda_stream)))
        st.synchronize()
        host = p.host_view()
        exp_host = before_host.clone()
        for g, h, s, n in segs:
            exp_host[h, l0:l1, :, :, s:s + n] = before_gpu[g, l0:l1, :, :, s:s + n]
        assert torch.equal(host, exp_host)
        # scatter back into different blocks, then compare
        segs2 = [((g + 7) % nb, h, s, n) for g, h, s, n in segs]
        before_gpu2 = p.gpu_view().cpu().clone()
        lib.check(lib.lib.tf_kv_scatter_h2d(p.handle, _segs(lib, segs2), len(segs2), l0, l1, engine,
                                            C.c_void_p(st.cuda_stream)))
        st.synchronize()
        exp_gpu = before_gpu2.clone()
        for g, h, s, n in segs2:
            exp_gpu[g, l0:l1, :, :, s:s + n] = exp_host[h, l0:l1, :, :, s:s + n]
        assert torch.equal(p.gpu_view().cpu(), exp_gpu)
    p.close()


def test_swap_rejects_bad_segments(cuda):
    lib = _lib()
    p = _pool(cuda, 4, 4, 2, 2, 64)
    with pytest.raises(ValueError):
        lib.check(lib.lib.tf_kv_gather_d2h(p.handle, _segs(lib, [(9, 0, 0, 4)]), 1, 0, 2, 0, None))
    with pytest.raises(ValueError):
        lib.check(lib.lib.tf_kv_gather_d2h(p.handle, _segs(lib, [(0, 0, 10, 8)]), 1, 0, 2, 0, None))
    with pytest.raises(ValueError):
        lib.check(lib.lib.tf_kv_scatter_h2d(p.handle, _segs(lib, [(0, 0, 0, 4)]), 1, 1, 1, 0, None))
    lib.check(lib.lib.tf_kv_gather_d2h(p.handle, _segs(lib, []), 0, 0, 2, 0, None))  # empty is a no-op
    p.close()


_RNG = np.random.default_rng(5)
# (contexts, layers, kv heads, q heads, head_dim, layer): C2 shapes (Llama3-8B
# 32/8 hd128; Qwen2.5-32B TP=1 40/8) at batch 1 / 64 / 128 / 130 with ragged
# 1-3000 contexts, block-edge contexts, the C1 tiny decoder (4/2 hd64)
ATTN_CASES = {
    "llama_b1": ([2049], 32, 8, 32, 128, 31),
    "llama_edges": ([1, 15, 16, 17, 100, 700, 2049, 4000], 32, 8, 32, 128, 5),
    "llama_b64_ragged": ([int(x) for x in _RNG.integers(1, 3000, 64)], 32, 8, 32, 128, 7),
    "llama_b128_c2": ([int(x) for x in _RNG.integers(300, 900, 128)], 4, 8, 32, 128, 3),
    "llama_b130_ragged": ([int(x) for x in _RNG.integers(1, 3000, 130)], 4, 8, 32, 128, 2),
    "qwen_g5": ([17, 900, 4096, 1, 2500], 4, 8, 40, 128, 1),
    "tiny_hd64": ([3, 64, 200, 513, 1000], 2, 2, 4, 64, 1),
    "g8": ([33, 1000], 2, 4, 32, 128, 0),
}


@pytest.mark.parametrize("impl", [5, 3])
@pytest.mark.parametrize("name", list(ATTN_CASES))
def test_paged_attention_vs_fp32(cuda, impl, name):
    """Every row within 2e-2 of its own fp32 magnitude (attn_parity.py)."""
    from attn_parity import run

    ctx, L, H, HQ, D, layer = ATTN_CASES[name]
    r = run(ctx, L, H, HQ, D, layer, impl=impl)
    assert r <= 1.0, f"worst row error is {r:.2f}x the tolerance"


@pytest.mark.parametrize("impl", [5, 3])
def test_paged_attention_graph_plan_vs_fp32(cuda, impl):
    """The CUDA-graph decode plan: launch captured ONCE for a 128-row bucket
    with max_ctx = the pool maximum, padding rows on the scratch row; then the
    real rows / contexts / q change on the device and the graph is replayed
    (the workspace counters must self-reset between replays)."""
    from attn_parity import REL_TOL, launch, make_case, worst_ratio
    from paper_2510_02758_b200 import _lib as L_

    prev = L_.lib.tf_paged_decode_attn_impl(impl)
    try:
        rng = np.random.default_rng(11)
        ctx = [int(x) for x in rng.integers(1, 3000, 100)]
        case = make_case(cuda, ctx, 3, 8, 32, 128, seed=3, pad_to=128, map_ctx=3000)
        pool_max = 16 * 400  # the graphs plan for the pool's maximum context
        st = torch.cuda.Stream()
        out = torch.zeros_like(case["q"])
        ws_n = max(1, int(L_.lib.tf_paged_decode_attn_workspace(case["pool"].handle, 128, pool_max, 32)))
        ws = torch.zeros(ws_n, dtype=torch.uint8, device=cuda)
        with torch.cuda.stream(st):
            launch(case, 1, max_ctx=pool_max, out=out, ws=ws, stream=st)  # warm-up (attributes, tensor map)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            launch(case, 1, max_ctx=pool_max, out=out, ws=ws, stream=torch.cuda.current_stream())
        for rep in range(3):
            # new contexts (a different ragged batch) and new q, same buffers
            new = [int(x) for x in rng.integers(1, 3000, 100)]
            case["ctx"][:100].copy_(torch.tensor(new, dtype=torch.int32))
            case["q"].copy_((torch.randn_like(case["q"].float()) * 4).to(torch.bfloat16))
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            r = worst_ratio(case, 1, out)
            assert r <= 1.0, f"replay {rep}: worst row error {r:.2f}x the {REL_TOL} tolerance"
        case["pool"].close()
    finally:
        L_.lib.tf_paged_decode_attn_impl(prev)


@pytest.mark.parametrize("impl", [5, 3])
def test_paged_attention_parity_catches_a_dropped_split(cuda, impl):
    """The parity check can fail: with TF_ATTN_MUTATE=1 every (request, kv
    head) of >= 8 blocks ignores its last eighth (a lost split); the same
    check run in a subprocess must report a violation at C2 contexts."""
    import os
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, 'tests'); from attn_parity import run; "
            f"print(run([2049, 4000, 700, 1500], 4, 8, 32, 128, 2, impl={impl}))")
    env = dict(os.environ, TF_ATTN_MUTATE="1")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                         cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    assert res.returncode == 0, res.stderr[-2000:]
    ratio = float(res.stdout.strip().splitlines()[-1])
    assert ratio > 1.0, f"mutated kernel passed the parity check (ratio {ratio:.2f})"


@pytest.mark.parametrize("knob", ["TF_ATTN_TR=1", "TF_ATTN_BALANCED=1", "TF_ATTN_PF=2", "TF_ATTN_STAGES=3",
                                  "TF_ATTN_STAGES=2"])
def test_paged_attention_opt_in_variants_vs_fp32(cuda, knob):
    """The measured-but-not-default v3 variants (transposed inner loop,
    device-balanced split plan, L2 prefetch, forced ring depth) stay within
    the parity tolerance; each runs in a subprocess because the library reads
    its knobs once per process."""
    import os
    import subprocess
    import sys

    k, v = knob.split("=")
    code = ("import sys; sys.path.insert(0, 'tests'); from attn_parity import run; import numpy as np; "
            "rng = np.random.default_rng(9); "
            "print(max(run(c, 4, 8, 32, 128, 1, impl=3) for c in ("
            "[int(x) for x in rng.integers(1, 3000, 64)], [int(x) for x in rng.integers(200, 900, 128)], "
            "[1, 15, 16, 17, 2049, 4000])))")
    res = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **{k: v}), capture_output=True,
                         text=True, timeout=300, cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    assert res.returncode == 0, res.stderr[-2000:]
    ratio = float(res.stdout.strip().splitlines()[-1])
    assert ratio <= 1.0, f"{knob}: worst row error is {ratio:.2f}x the tolerance"


def test_paged_attention_workspace_reuse_is_deterministic(cuda):
    """The stream-K merge counters reset themselves: relaunching with the same
    workspace gives bit-identical outputs (merge order is fixed by slot)."""
    from attn_parity import launch, make_case

    ctx_list = [int(x) for x in np.random.default_rng(9).integers(1, 2500, 48)]
    case = make_case(cuda, ctx_list, 2, 8, 32, 128, seed=4)
    out0, ws = launch(case, 1, max_ctx=4096)
    outs = [out0.clone()]
    for _ in range(2):
        o, _ = launch(case, 1, max_ctx=4096, ws=ws)
        outs.append(o.clone())
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
    case["pool"].close()


def test_kv_append_writes_slots(cuda):
    lib = _lib()
    L, H, D = 2, 2, 64
    p = _pool(cuda, 8, 1, L, H, D)
    table = torch.tensor([[3, 5], [6, -1]], dtype=torch.int32, device=cuda)
    rows = torch.tensor([0, 0, 1], dtype=torch.int32, device=cuda)
    pos = torch.tensor([0, 17, 9], dtype=torch.int32, device=cuda)
    kv = torch.randint(-1000, 1000, (3, 2, H, D), dtype=torch.int16, device=cuda)
    lib.check(lib.lib.tf_kv_append(p.handle, C.c_void_p(table.data_ptr()), 2, C.c_void_p(rows.data_ptr()),
                                   C.c_void_p(pos.data_ptr()), 3, 1, C.c_void_p(kv[:, 0].data_ptr()),
                                   C.c_void_p(kv[:, 1].data_ptr()), 2 * H * D, None))
    torch.cuda.synchronize()
    g = p.gpu_view().cpu()
    kvc = kv.cpu()
    for i, (blk, slot) in enumerate([(3, 0), (5, 1), (6, 9)]):
        assert torch.equal(g[blk, 1, 0, :, slot], kvc[i, 0])
        assert torch.equal(g[blk, 1, 1, :, slot], kvc[i, 1])
    p.close()


@pytest.mark.parametrize("hq,hkv,D,n,wt", [(32, 8, 128, 128, False), (40, 8, 128, 5, False), (4, 2, 64, 300, False),
                                           (32, 8, 128, 7, True)])
def test_rope_kv_append_vs_torch(cuda, hq, hkv, D, n, wt):
    """Fused rotary + paged append: q rotated into q_out, k rotated and v copied
    into each token's pool slot (and the contiguous kv_out copy; with fused
    write-through also into the host block), against a torch fp32 rotary."""
    lib = _lib()
    L, layer = 3, 1
    nb = n // 16 + 4
    p = _pool(cuda, 2 * nb + 2, 2 * nb + 2, L, hkv, D)
    rows = torch.tensor([i % 2 for i in range(n)], dtype=torch.int32, device=cuda)
    posl = [i // 2 + 3 * (i % 2) for i in range(n)]
    pos = torch.tensor(posl, dtype=torch.int32, device=cuda)
    nlb = max(posl) // 16 + 1
    table = torch.tensor([list(range(nlb)), list(range(nb, nb + nlb))], dtype=torch.int32, device=cuda)
    htable = torch.tensor([list(range(nlb, 2 * nlb)), list(range(0, nlb))], dtype=torch.int32, device=cuda)
    heads = hq + 2 * hkv
    qkv = torch.randn(n, heads, D, device=cuda).to(torch.bfloat16)
    inv = 1.0 / (500000.0 ** (torch.arange(0, D, 2, device=cuda, dtype=torch.float32) / D))
    q_out = torch.empty(n, hq, D, device=cuda, dtype=torch.bfloat16)
    kv_out = torch.empty(2, n, hkv, D, device=cuda, dtype=torch.bfloat16)
    if wt:
        lib.check(lib.lib.tf_rope_kv_append_wt(p.handle, C.c_void_p(table.data_ptr()), C.c_void_p(htable.data_ptr()),
                                               nlb, C.c_void_p(rows.data_ptr()), C.c_void_p(pos.data_ptr()), n, layer,
                                               C.c_void_p(qkv.data_ptr()), hq, C.c_void_p(inv.data_ptr()),
                                               C.c_void_p(q_out.data_ptr()), C.c_void_p(kv_out.data_ptr()), None))
    else:
        lib.check(lib.lib.tf_rope_kv_append(p.handle, C.c_void_p(table.data_ptr()), nlb, C.c_void_p(rows.data_ptr()),
                                            C.c_void_p(pos.data_ptr()), n, layer, C.c_void_p(qkv.data_ptr()), hq,
                                            C.c_void_p(inv.data_ptr()), C.c_void_p(q_out.data_ptr()),
                                            C.c_void_p(kv_out.data_ptr()), None))
    torch.cuda.synchronize()

    def rope(x):  # interleaved pairs, fp32
        ang = pos.float()[:, None, None] * inv[None, None, :]
        x1, x2 = x[..., 0::2].float(), x[..., 1::2].float()
        out = torch.empty_like(x, dtype=torch.float32)
        out[..., 0::2] = x1 * ang.cos() - x2 * ang.sin()
        out[..., 1::2] = x1 * ang.sin() + x2 * ang.cos()
        return out

    q_ref = rope(qkv[:, :hq])
    k_ref = rope(qkv[:, hq:hq + hkv])
    v_ref = qkv[:, hq + hkv:]
    tol = lambda r: 2 ** -7 * r.abs() + 2 ** -12  # noqa: E731  (bf16 rounding + sincos ulps)
    assert ((q_out.float() - q_ref).abs() <= tol(q_ref)).all()
    assert ((kv_out[0].float() - k_ref).abs() <= tol(k_ref)).all()
    assert torch.equal(kv_out[1], v_ref)
    g = p.gpu_view().view(torch.bfloat16)
    hv = p.host_view().view(torch.bfloat16)
    for i in range(n):
        r, ps = int(rows[i]), posl[i]
        blk = int(table[r, ps // 16])
        assert torch.equal(g[blk, layer, 0, :, ps % 16], kv_out[0, i])
        assert torch.equal(g[blk, layer, 1, :, ps % 16], kv_out[1, i])
        if wt:
            hb = int(htable[r, ps // 16])
            assert torch.equal(hv[hb, layer, 0, :, ps % 16], kv_out[0, i].cpu())
            assert torch.equal(hv[hb, layer, 1, :, ps % 16], kv_out[1, i].cpu())
    p.close()


@pytest.mark.parametrize("rows,dim", [(1, 256), (37, 4096), (128, 5120), (3000, 4096)])
def test_rmsnorm_vs_torch(cuda, rows, dim):
    import torch.nn.functional as F

    lib = _lib()
    x = (torch.randn(rows, dim, device=cuda) * 3).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(dim, device=cuda)).to(torch.bfloat16)
    y = torch.empty_like(x)
    lib.check(lib.lib.tf_rmsnorm(C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr()),
                                 rows, dim, 1e-5, None))
    torch.cuda.synchronize()
    ref = F.rms_norm(x.float(), (dim,), w.float(), 1e-5)
    # bf16 output: within 2 bf16 ulps of the fp32 reference
    assert ((y.float() - ref).abs() <= 2 ** -6 * ref.abs() + 1e-3).all()


@pytest.mark.parametrize("rows,dim", [(1, 256), (64, 4096), (128, 5120), (300, 8192)])
def test_residual_rmsnorm_bit_exact(cuda, rows, dim):
    """x += y (one bf16 rounding of the fp32 sum), h = rmsnorm(x) * w: the new
    residual equals the fp32 definition bit for bit and h equals tf_rmsnorm of it."""
    lib = _lib()
    x = (torch.randn(rows, dim, device=cuda) * 3).to(torch.bfloat16)
    y = torch.randn(rows, dim, device=cuda).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(dim, device=cuda)).to(torch.bfloat16)
    x_ref = (x.float() + y.float()).to(torch.bfloat16)
    h = torch.empty_like(x)
    lib.check(lib.lib.tf_residual_rmsnorm(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                          C.c_void_p(w.data_ptr()), C.c_void_p(h.data_ptr()), rows, dim, 1e-5, None))
    h_ref = torch.empty_like(x)
    lib.check(lib.lib.tf_rmsnorm(C.c_void_p(x_ref.data_ptr()), C.c_void_p(w.data_ptr()),
                                 C.c_void_p(h_ref.data_ptr()), rows, dim, 1e-5, None))
    torch.cuda.synchronize()
    assert torch.equal(x.view(torch.int16), x_ref.view(torch.int16))
    assert torch.equal(h.view(torch.int16), h_ref.view(torch.int16))


@pytest.mark.parametrize("rows,ffn", [(1, 688), (64, 14336), (200, 3456), (70000, 16)])
def test_silu_mul_vs_torch(cuda, rows, ffn):
    import torch.nn.functional as F

    lib = _lib()
    gu = (torch.randn(rows, 2 * ffn, device=cuda) * 2).to(torch.bfloat16)
    y = torch.empty(rows, ffn, device=cuda, dtype=torch.bfloat16)
    lib.check(lib.lib.tf_silu_mul(C.c_void_p(gu.data_ptr()), C.c_void_p(y.data_ptr()), rows, ffn, None))
    torch.cuda.synchronize()
    g, u = gu.float().chunk(2, dim=-1)
    ref = F.silu(g) * u
    assert ((y.float() - ref).abs() <= 2 ** -6 * ref.abs() + 1e-3).all()


def test_launch_counter_counts_library_kernels(cuda):
    """tf_launch_count (the bench's gpu_launches) advances by one per kernel
    the library launches."""
    lib = _lib()
    x = torch.randn(4, 256, device=cuda).to(torch.bfloat16)
    w = torch.ones(256, device=cuda).to(torch.bfloat16)
    y = torch.empty_like(x)
    c0 = lib.lib.tf_launch_count()
    for _ in range(3):
        lib.check(lib.lib.tf_rmsnorm(C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr()),
                                     4, 256, 1e-5, None))
    torch.cuda.synchronize()
    assert lib.lib.tf_launch_count() - c0 == 3

"""Paged decode attention vs an fp32 reference (helper of test_kernels_gpu.py;
also run as a subprocess under TF_ATTN_MUTATE=1 to prove the check fails).

Tolerance (north star: "within a stated bf16 tolerance, e.g. max-abs 2e-2
relative to fp32"): for every (request, q head) row,
    max |out - ref| <= 2e-2 * max |ref| + 2**-10
i.e. 2% of the row's own magnitude plus a bf16-rounding floor.  Inputs are
scaled so the softmax is peaked (q ~ 4 N(0,1), K, V ~ 0.5 N(0,1)): long
contexts then still have O(0.1-1) outputs, and dropping any eighth of a
context moves a row by 10-50% of its magnitude.

Reference: tokensim/costs.py:45-59 is the cost the kernel replaces; the
semantics are the plain softmax(q K^T / sqrt(d)) V over the request's
paged positions [0, ctx).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

REL_TOL = 2e-2
ABS_FLOOR = 2.0 ** -10


def _lib():
    from paper_2510_02758_b200 import _lib

    return _lib


def make_case(cuda, ctx_list, L, H, HQ, D, seed=0, pad_to=None, map_ctx=0):
    """Pool + tables + q for a batch with the given contexts.  ``pad_to``:
    append padding rows (the CUDA-graph bucket layout: they point at a
    scratch table row whose one block is mapped, ctx 1).  ``map_ctx``: map
    at least this many positions per row (so contexts can later grow)."""
    from paper_2510_02758_b200.dataplane import KvPool

    B = len(ctx_list)
    nblk_req = [(max(c, map_ctx) + 15) // 16 for c in ctx_list]
    nb = sum(nblk_req) + 2
    p = KvPool(nb, 1, L, H, D, device=cuda)
    g = torch.Generator(device=cuda).manual_seed(seed)
    kv = (torch.randn(p.gpu.numel(), device=cuda, generator=g) * 0.5).to(torch.bfloat16).view(torch.int16)
    p.gpu.copy_(kv)
    maxlb = max(nblk_req)
    perm = np.random.default_rng(seed + 1).permutation(nb)
    n_rows = B + 1
    table = np.full((n_rows, maxlb), -1, np.int32)
    k = 0
    for b in range(B):
        table[b, : nblk_req[b]] = perm[k:k + nblk_req[b]]
        k += nblk_req[b]
    scratch = B
    table[scratch, :] = perm[k]  # scratch row: one block, every logical block
    rows = list(range(B))
    ctx = list(ctx_list)
    if pad_to is not None and pad_to > B:
        rows += [scratch] * (pad_to - B)
        ctx += [1] * (pad_to - B)
    Bp = len(rows)
    q = (torch.randn(Bp, HQ, D, device=cuda, generator=g) * 4.0).to(torch.bfloat16)
    return {"pool": p, "table": torch.from_numpy(table).to(cuda), "maxlb": maxlb,
            "rows": torch.tensor(rows, dtype=torch.int32, device=cuda),
            "ctx": torch.tensor(ctx, dtype=torch.int32, device=cuda), "q": q, "B": B, "Bp": Bp,
            "L": L, "H": H, "HQ": HQ, "D": D}


def launch(case, layer, max_ctx=None, out=None, ws=None, stream=None):
    lib = _lib()
    p, HQ, D, Bp = case["pool"], case["HQ"], case["D"], case["Bp"]
    max_ctx = max_ctx or int(case["ctx"].max().item())
    if out is None:
        out = torch.empty_like(case["q"])
    if ws is None:
        ws_n = max(1, int(lib.lib.tf_paged_decode_attn_workspace(p.handle, Bp, max_ctx, HQ)))
        ws = torch.zeros(ws_n, dtype=torch.uint8, device=case["q"].device)
    lib.check(lib.lib.tf_paged_decode_attn(
        p.handle, C.c_void_p(case["q"].data_ptr()), C.c_void_p(case["table"].data_ptr()), case["maxlb"],
        C.c_void_p(case["rows"].data_ptr()), C.c_void_p(case["ctx"].data_ptr()), Bp, max_ctx, layer, HQ,
        1.0 / D ** 0.5, C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(),
        C.c_void_p(0 if stream is None else stream.cuda_stream)), "tf_paged_decode_attn")
    return out, ws


def reference(case, layer, b):
    """fp32 (float64 softmax) attention of request row b -> [HQ][D]."""
    p, H, HQ, D = case["pool"], case["H"], case["HQ"], case["D"]
    G = HQ // H
    pool = p.gpu_view().view(torch.bfloat16)
    row = int(case["rows"][b])
    c = int(case["ctx"][b])
    t = torch.arange(c, device=pool.device)
    blk = case["table"][row][(t // 16).long()].long()
    kk = pool[blk, layer, 0, :, (t % 16).long()].float()  # [T][H][D]
    vv = pool[blk, layer, 1, :, (t % 16).long()].float()
    qf = case["q"][b].float().view(H, G, D)
    s = torch.einsum("hgd,thd->hgt", qf, kk) / D ** 0.5
    pr = torch.softmax(s.double(), -1).float()
    return torch.einsum("hgt,thd->hgd", pr, vv).reshape(HQ, D)


def worst_ratio(case, layer, out, rows=None):
    """max over rows of  max|out - ref| / (REL_TOL * max|ref| + ABS_FLOOR)  (<= 1 passes)."""
    worst = 0.0
    for b in (rows if rows is not None else range(case["B"])):
        ref = reference(case, layer, b)
        err = (out[b].float() - ref).abs().amax(-1)
        lim = REL_TOL * ref.abs().amax(-1) + ABS_FLOOR
        worst = max(worst, float((err / lim).max()))
    return worst


def run(ctx_list, L, H, HQ, D, layer, impl=None, pad_to=None, max_ctx=None, seed=0):
    """-> worst ratio for one launch (used by the mutation subprocess)."""
    lib = _lib()
    prev = lib.lib.tf_paged_decode_attn_impl(impl if impl is not None else -1)
    try:
        case = make_case("cuda", ctx_list, L, H, HQ, D, seed=seed, pad_to=pad_to)
        out, _ = launch(case, layer, max_ctx=max_ctx)
        torch.cuda.synchronize()
        r = worst_ratio(case, layer, out)
        case["pool"].close()
        return r
    finally:
        lib.lib.tf_paged_decode_attn_impl(prev)

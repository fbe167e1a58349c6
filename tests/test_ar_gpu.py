"""C4 data path: the peer-memory all-reduce fused with the residual add and
the next RMSNorm (csrc/tf_ar.cu, tp.PeerAllReduce).

* same-process ranks (one stream each, peers linked by pointer): bit-exact
  against the fp32 definition x' = bf16(x + sum_p part_p) and against
  tf_rmsnorm(x'); every rank ends with identical x; CUDA-graph replays
  advance the device-resident barrier epochs correctly;
* the TP=2 decoder on that path equals the TP=2 decoder on the plain
  all-reduce path, and stays within the logits tolerance of TP=1;
* two PROCESSES on one GPU exchanging CUDA IPC handles over gloo (the code
  path of a multi-GPU run; there the peers are NVLink P2P mappings).
"""
import ctypes as C
import threading

import pytest

pytestmark = pytest.mark.gpu


def _ranks(world, cap, cuda):
    from paper_2510_02758_b200.tp import PeerAllReduce

    # same-process ranks share the GPU: a few CTAs each, so a waiting rank
    # never holds the SMs another rank's GEMM needs
    ars = [PeerAllReduce(r, world, cap, device=cuda, max_ctas=8) for r in range(world)]
    PeerAllReduce.link(ars)
    return ars


def _ref(x, parts, gamma, eps):
    import torch

    s = parts[0].float()
    for p in parts[1:]:
        s = s + p.float()
    xn = (s + x.float()).to(torch.bfloat16)
    return xn


def _tf_rms(x, gamma, eps):
    import torch

    from paper_2510_02758_b200._lib import check, lib

    y = torch.empty_like(x)
    check(lib.tf_rmsnorm(C.c_void_p(x.data_ptr()), C.c_void_p(gamma.data_ptr()), C.c_void_p(y.data_ptr()),
                         x.shape[0], x.shape[1], eps, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return y


def _run_ranks(ars, fn):
    """fn(rank) on one thread + stream per rank (kernels of different ranks
    must be able to run concurrently: they wait for each other)."""
    import torch

    errs = []

    def go(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                fn(r, st)
            st.synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    th = [threading.Thread(target=go, args=(r,)) for r in range(len(ars))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.parametrize("world,rows,dim", [(2, 1, 256), (2, 128, 4096), (4, 64, 5120), (8, 24, 5120),
                                            (2, 300, 5120), (2, 17, 8192)])
def test_fused_allreduce_residual_rmsnorm_bit_exact(cuda, world, rows, dim):
    import torch

    eps = 1e-6
    ars = _ranks(world, rows * dim * 2, cuda)
    g = torch.Generator(device=cuda).manual_seed(rows + dim + world)
    parts = [torch.randn(rows, dim, device=cuda, generator=g).to(torch.bfloat16) for _ in range(world)]
    x0 = torch.randn(rows, dim, device=cuda, generator=g).to(torch.bfloat16)
    gamma = (1.0 + 0.1 * torch.randn(dim, device=cuda, generator=g)).to(torch.bfloat16)
    xs = [x0.clone() for _ in range(world)]
    hs = [torch.empty_like(x0) for _ in range(world)]
    for r in range(world):
        ars[r].partial(rows, dim).copy_(parts[r])
    torch.cuda.synchronize()
    _run_ranks(ars, lambda r, st: ars[r].residual_rmsnorm(xs[r], gamma, hs[r], eps, st))
    torch.cuda.synchronize()
    ref = _ref(x0, parts, gamma, eps)
    href = _tf_rms(ref, gamma, eps)
    for r in range(world):
        assert ars[r].status() == 0
        assert torch.equal(xs[r].view(torch.int16), ref.view(torch.int16)), f"rank {r}: residual differs"
        assert torch.equal(hs[r].view(torch.int16), href.view(torch.int16)), f"rank {r}: norm differs"
    # and the norm itself is the fp32 definition (bf16 rounding of x*rsqrt, then * gamma)
    xf = ref.float()
    hf = (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(torch.bfloat16).float() * gamma.float()
    assert torch.allclose(hs[0].float(), hf, rtol=1e-2, atol=1e-2)
    for a in ars:
        a.close()


def test_plain_sum_mode(cuda):
    import torch

    ars = _ranks(2, 64 * 512 * 2, cuda)
    parts = [torch.randn(64, 512, device=cuda).to(torch.bfloat16) for _ in range(2)]
    for r in range(2):
        ars[r].partial(64, 512).copy_(parts[r])
    outs = [torch.empty(64, 512, device=cuda, dtype=torch.bfloat16) for _ in range(2)]
    torch.cuda.synchronize()
    from paper_2510_02758_b200._lib import check, lib

    def go(r, st):
        check(lib.tf_ar_residual_rmsnorm(ars[r].handle, None, None, C.c_void_p(outs[r].data_ptr()), 64, 512,
                                         1e-6, C.c_void_p(st.cuda_stream)))

    _run_ranks(ars, go)
    ref = (parts[0].float() + parts[1].float()).to(torch.bfloat16)
    assert torch.equal(outs[0], ref) and torch.equal(outs[1], ref)


def test_rejects_bad_arguments(cuda):
    import torch

    from paper_2510_02758_b200._lib import check, lib

    ars = _ranks(2, 1024, cuda)
    x = torch.zeros(4, 256, device=cuda, dtype=torch.bfloat16)
    with pytest.raises(ValueError):  # 4 x 256 x 2 B > 1024-byte buffer
        ars[0].residual_rmsnorm(x, None, x, 1e-6)
    with pytest.raises(ValueError):
        check(lib.tf_ar_residual_rmsnorm(ars[0].handle, C.c_void_p(x.data_ptr()), None, None, 1, 12, 1e-6, None))
    with pytest.raises(ValueError):
        check(lib.tf_ar_create(2, 2, 1024, 0, C.byref(C.c_int64())))
    with pytest.raises(ValueError):
        check(lib.tf_ar_create(0, 9, 1024, 0, C.byref(C.c_int64())))
    with pytest.raises(ValueError):
        check(lib.tf_ar_create(0, 2, 1024, 149, C.byref(C.c_int64())))


def test_graph_replays_advance_the_barrier(cuda):
    """Three fused calls captured per rank; five replays with fresh partials
    must each give the reference result (the epochs live on the device)."""
    import torch

    world, rows, dim, eps = 2, 48, 1024, 1e-5
    ars = _ranks(world, rows * dim * 2, cuda)
    gamma = torch.ones(dim, device=cuda, dtype=torch.bfloat16)
    xs = [torch.zeros(rows, dim, device=cuda, dtype=torch.bfloat16) for _ in range(world)]
    hs = [torch.empty_like(xs[0]) for _ in range(world)]
    src = [torch.zeros(rows, dim, device=cuda, dtype=torch.bfloat16) for _ in range(world)]
    graphs = [torch.cuda.CUDAGraph() for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    for r in range(world):  # capture (no launch happens during capture)
        with torch.cuda.graph(graphs[r], stream=streams[r]):
            for _ in range(3):
                ars[r].partial(rows, dim).copy_(src[r])
                ars[r].residual_rmsnorm(xs[r], gamma, hs[r], eps, torch.cuda.current_stream())
    torch.cuda.synchronize()
    for it in range(5):
        x0 = torch.randn(rows, dim, device=cuda).to(torch.bfloat16)
        ps = [torch.randn(rows, dim, device=cuda).to(torch.bfloat16) for _ in range(world)]
        for r in range(world):
            xs[r].copy_(x0)
            src[r].copy_(ps[r])
        torch.cuda.synchronize()
        _run_ranks(ars, lambda r, st: (st.wait_stream(streams[r]), graphs[r].replay()))
        torch.cuda.synchronize()
        ref = x0
        for _ in range(3):
            ref = _ref(ref, ps, gamma, eps)
        for r in range(world):
            assert torch.equal(xs[r], ref), f"replay {it} rank {r}"
            assert torch.equal(hs[r], _tf_rms(ref, gamma, eps))
    assert all(a.status() == 0 for a in ars)


def test_tp2_decoder_on_peer_path(cuda):
    """The TP=2 decoder (two threads, one stream each) on the fused peer path
    computes the same KV as on the plain all-reduce path and its logits stay
    within 2e-2 * max|l| of TP=1."""
    import torch
    from test_tp_gpu import ThreadTp, _setup

    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200.tp import PeerAllReduce

    shape = configs.TINY
    n_req, nlb = 4, 5
    seqs = [(i, torch.randint(0, shape.vocab, (30 + 9 * i,), generator=torch.Generator().manual_seed(i)), 0)
            for i in range(n_req)]
    m1, dp1, pool1 = _setup(cuda, shape, None, n_req, nlb)
    m1.keep_logits = True
    with torch.cuda.stream(dp1.s_compute):
        m1._prefill_batch(dp1, seqs, dp1.s_compute)
    torch.cuda.synchronize()

    def tp2(peer):
        shared = {"buf": [None, None], "bar": threading.Barrier(2)}
        shards = []
        ars = ([PeerAllReduce(r, 2, 4096 * shape.hidden * 2, device=cuda, max_ctas=8) for r in range(2)]
               if peer else None)
        if peer:
            PeerAllReduce.link(ars)
        for r in range(2):
            t = ThreadTp(r, 2, shared)
            t.ar = ars[r] if peer else None
            shards.append(_setup(cuda, shape, t, n_req, nlb))
        outs = [None, None]

        def run(r):
            m, dp, _ = shards[r]
            m.keep_logits = True
            with torch.cuda.stream(dp.s_compute):
                outs[r] = m._prefill_batch(dp, seqs, dp.s_compute)
            dp.s_compute.synchronize()

        th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        if peer:
            assert all(a.status() == 0 for a in ars)
        return shards, outs

    sp, op = tp2(True)
    sn, on = tp2(False)
    assert torch.equal(op[0], op[1])
    l1 = m1.last_logits.float()
    for r in range(2):
        lp = sp[r][0].last_logits.float()
        assert torch.equal(lp, sp[0][0].last_logits.float()), "ranks disagree on the peer path"
        err = (lp - l1).abs().amax(-1)
        assert bool((err <= 2e-2 * l1.abs().amax(-1) + 2.0 ** -8).all()), err.tolist()
        # peer path vs plain all-reduce path: same partition, different (but
        # both fp32) residual order -> KV equal within bf16 rounding
        a = sp[r][2].gpu_view().view(torch.bfloat16).float()
        b = sn[r][2].gpu_view().view(torch.bfloat16).float()
        used = n_req * nlb
        assert (a[:used] - b[:used]).abs().max().item() <= 2e-2 * max(1.0, b[:used].abs().max().item())


def _ipc_worker(rank, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2510_02758_b200.tp import PeerAllReduce

    rows, dim, eps = 64, 1024, 1e-6
    ar = PeerAllReduce.from_group(rank, 2, rows * dim * 2, device=torch.device("cuda", 0), max_ctas=8)
    gamma = torch.ones(dim, device="cuda", dtype=torch.bfloat16)
    res = []
    for it in range(3):
        g = torch.Generator(device="cuda").manual_seed(100 * it + rank)
        ar.partial(rows, dim).copy_(torch.randn(rows, dim, device="cuda", generator=g).to(torch.bfloat16))
        x = torch.full((rows, dim), 0.5, device="cuda", dtype=torch.bfloat16)
        h = torch.empty_like(x)
        torch.cuda.synchronize()
        dist.barrier()
        ar.residual_rmsnorm(x, gamma, h, eps)
        torch.cuda.synchronize()
        res.append(x.view(torch.int16).cpu().numpy())  # plain arrays: no fd-shared tensors through the queue
        dist.barrier()
    q.put((rank, ar.status(), res))
    dist.barrier()
    ar.close()
    dist.destroy_process_group()


def test_two_processes_over_cuda_ipc(cuda):
    import socket

    import torch
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (st, res)) for r, st, res in (q.get(timeout=300), q.get(timeout=300)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0][0] == 0 and got[1][0] == 0, "a barrier timed out"
    for it in range(3):
        parts = []
        for r in range(2):
            g = torch.Generator(device="cuda").manual_seed(100 * it + r)
            parts.append(torch.randn(64, 1024, device="cuda", generator=g).to(torch.bfloat16))
        ref = _ref(torch.full((64, 1024), 0.5, device="cuda", dtype=torch.bfloat16), parts, None, 0)
        ref = ref.view(torch.int16).cpu().numpy()
        assert (got[0][1][it] == ref).all() and (got[1][1][it] == ref).all()

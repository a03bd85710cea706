"""Kernel parity on the B200 through the C ABI (mlt_*).

* GEMM / expert FFN / RMSNorm / attention: against a plain PyTorch fp32
  reference of the same op on the same bf16 inputs (tolerances stated per
  test; only summation order differs).
* Router: BIT-EXACT against the CPU oracle (oracle/oracle_numerics.c
  orc_router) on identical bf16 inputs — logits, top-k indices and the
  stable permutation (BASELINE.json correctness item 1).
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2411_11217_b200 import capi  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(scope="module")
def K():
    return capi.load_kernels()


def ptr(t):
    return C.c_void_p(t.data_ptr())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def rand_bf16(*shape, scale=1.0, gen=None):
    return (torch.randn(*shape, generator=gen) * scale).to(torch.bfloat16)


def unif_bf16(*shape, scale=1.0, gen=None):
    """uniform(-sqrt3 s, sqrt3 s): the runtime's synthetic-weight distribution
    (the 3-bit code, codec 4, falls back to raw blocks on Gaussian tiles)."""
    return ((torch.rand(*shape, generator=gen) * 2 - 1) * (3 ** 0.5 * scale)).to(torch.bfloat16)


def bf16_bits(t):  # torch bf16 -> numpy uint16 view
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def pack_weight_dev(K, w_bf16):
    """Host-pack a [M, K] bf16 weight and upload; returns (device buffer, block pointers)."""
    M, Kd = w_bf16.shape
    src = bf16_bits(w_bf16.cpu())
    dst = np.empty_like(src)
    K.pack_weight(src.ctypes.data_as(C.c_void_p), M, Kd, dst.ctypes.data_as(C.c_void_p))
    dev = torch.from_numpy(dst.view(np.int16).copy()).cuda()
    blocks = [dev.data_ptr() + rb * 128 * Kd * 2 for rb in range(M // 128)]
    return dev, blocks


def table(ptr_lists):
    flat = [p for lst in ptr_lists for p in lst]
    return torch.tensor(flat, dtype=torch.int64, device="cuda")


def pack_rows_dev(K, x_bf16, R):
    T, Kd = x_bf16.shape
    out = torch.zeros(R * Kd, dtype=torch.int16, device="cuda")
    xd = x_bf16.cuda().contiguous()
    K.pack_rows(ptr(xd), Kd, T, Kd, ptr(out), R, stream())
    return out


@pytest.mark.parametrize("T,M,Kd,n_cap", [(1, 128, 64, 16), (16, 256, 512, 16), (37, 384, 1024, 64),
                                          (64, 256, 4096, 64), (200, 128, 256, 208),
                                          (256, 512, 1024, 256), (300, 256, 512, 128)])
def test_dense_gemm_matches_torch(K, T, M, Kd, n_cap):
    g = torch.Generator().manual_seed(T * 7 + M)
    w = rand_bf16(M, Kd, scale=Kd ** -0.5, gen=g)
    x = rand_bf16(T, Kd, gen=g)
    R = (T + 15) // 16 * 16
    wdev, blocks = pack_weight_dev(K, w)
    tab = table([blocks])
    xp = pack_rows_dev(K, x, R)
    res = torch.randn(T, M, device="cuda")
    out = torch.zeros(R, M, device="cuda")
    a = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=1, RB=M // 128, K=Kd, b=xp.data_ptr(),
                      R=R, b_off=None, b_cnt=None, rows_dense=T, n_cap=n_cap, epi=0, alpha=1.0,
                      out_f32=out.data_ptr(), ldo=M, residual=res.data_ptr(), ldr=M)
    K.gemm(C.byref(a), stream())
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T + res.cpu()
    err = (out[:T].cpu() - ref).abs().max().item()
    assert err <= 2e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("T,M,Kd,splits,chunks,n_cap", [(64, 384, 1024, 3, 1, 64),
                                                         (256, 256, 4096, 4, 1, 256),
                                                         (40, 128, 512, 8, 3, 16)])
def test_split_k_and_chunked_gemm(K, T, M, Kd, splits, chunks, n_cap):
    """Split-K partials (summed by the consumer) and N-chunked tiles."""
    g = torch.Generator().manual_seed(T + splits)
    w = rand_bf16(M, Kd, scale=Kd ** -0.5, gen=g)
    x = rand_bf16(T, Kd, gen=g)
    R = (T + 15) // 16 * 16
    wdev, blocks = pack_weight_dev(K, w)
    tab = table([blocks])
    xp = pack_rows_dev(K, x, R)
    parts = torch.zeros(splits, R, M, device="cuda")
    a = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=1, RB=M // 128, K=Kd, b=xp.data_ptr(),
                      R=R, rows_dense=T, n_cap=n_cap, epi=0, alpha=1.0, out_f32=parts.data_ptr(),
                      ldo=M, n_chunks=chunks, k_splits=splits, split_stride=R * M)
    K.gemm(C.byref(a), stream())
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T
    got = parts.sum(0)[:T].cpu()
    assert (got - ref).abs().max().item() <= 2e-3 * max(1.0, ref.abs().max().item())


def _expert_setup(T, H, Fd, E, Kk, seed, uniform=False):
    g = torch.Generator().manual_seed(seed)
    hn = rand_bf16(T, H, gen=g)
    wf = unif_bf16 if uniform else rand_bf16
    w1 = [wf(Fd, H, scale=H ** -0.5, gen=g) for _ in range(E)]
    w3 = [wf(Fd, H, scale=H ** -0.5, gen=g) for _ in range(E)]
    w2 = [wf(H, Fd, scale=Fd ** -0.5, gen=g) for _ in range(E)]
    wr = rand_bf16(E, H, scale=H ** -0.5, gen=g)
    return hn, w1, w3, w2, wr


@pytest.mark.parametrize("T,H,Fd,E,Kk,n_cap", [(4, 256, 384, 8, 2, 16), (64, 512, 768, 8, 2, 64),
                                               (256, 512, 256, 8, 2, 256), (33, 256, 256, 16, 4, 32)])
def test_router_permute_expert_ffn(K, T, H, Fd, E, Kk, n_cap):
    from oracle import bind as orc
    hn, w1, w3, w2, wr = _expert_setup(T, H, Fd, E, Kk, seed=T + H)
    hn_d, wr_d = hn.cuda(), wr.cuda()
    logits = torch.zeros(T, E, device="cuda")
    idx = torch.zeros(T, Kk, dtype=torch.int32, device="cuda")
    wts = torch.zeros(T, Kk, device="cuda")
    K.router_topk(None, None, 0.0, ptr(hn_d), ptr(wr_d), T, H, E, Kk, None, ptr(logits), ptr(idx),
                  ptr(wts), stream())
    R = T * Kk + 16 * E
    R = (R + 15) // 16 * 16
    cnt = torch.zeros(E, dtype=torch.int32, device="cuda")
    off = torch.zeros(E + 1, dtype=torch.int32, device="cuda")
    perm = torch.zeros(R, dtype=torch.int32, device="cuda")
    inv = torch.zeros(T * Kk, dtype=torch.int32, device="cuda")
    xp = torch.zeros(R * H, dtype=torch.int16, device="cuda")
    K.moe_permute(ptr(idx), ptr(hn_d), T, H, E, Kk, ptr(cnt), ptr(off), ptr(perm), ptr(inv),
                  ptr(xp), R, stream())
    torch.cuda.synchronize()

    # --- bit-exact router vs the CPU oracle on identical bf16 inputs ---
    o_log, o_idx, o_w, o_perm, o_off = orc.router(bf16_bits(hn), bf16_bits(wr), Kk)
    assert np.array_equal(logits.cpu().numpy().view(np.uint32), o_log.view(np.uint32))
    assert np.array_equal(idx.cpu().numpy(), o_idx)
    assert np.allclose(wts.cpu().numpy(), o_w, rtol=1e-6, atol=1e-7)
    c = cnt.cpu().numpy()
    assert np.array_equal(np.concatenate([[0], np.cumsum(c)]), o_off)
    offs, pm = off.cpu().numpy(), perm.cpu().numpy()
    unpadded = np.concatenate([pm[offs[e]:offs[e] + c[e]] for e in range(E)])
    assert np.array_equal(unpadded, o_perm)
    iv = inv.cpu().numpy()
    assert all(pm[iv[i]] == i for i in range(T * Kk))

    # --- expert FFN (gate/up + SiLU fused, down) + combine vs torch fp32 ---
    wd = []
    b13 = [[], []]
    b2 = []
    for e in range(E):
        d1, p1 = pack_weight_dev(K, w1[e])
        d3, p3 = pack_weight_dev(K, w3[e])
        d2, p2 = pack_weight_dev(K, w2[e])
        wd += [d1, d3, d2]
        b13[0] += p1
        b13[1] += p3
        b2 += p2
    t13, t2 = table(b13), table([b2])
    inter = torch.zeros(R * Fd, dtype=torch.int16, device="cuda")
    y = torch.zeros(R, H, device="cuda")
    h = torch.randn(T, H, device="cuda")
    xo = torch.zeros(T, H, device="cuda")
    K.expert_ffn(ptr(xp), R, ptr(cnt), ptr(off), ptr(t13), ptr(t2), E, H, Fd, n_cap, ptr(inter),
                 ptr(y), ptr(inv), ptr(wts), ptr(h), T, Kk, ptr(xo), stream())
    torch.cuda.synchronize()
    ref = h.cpu().clone()
    hnf = hn.float()
    for t in range(T):
        for s in range(Kk):
            e = int(o_idx[t, s])
            a = torch.nn.functional.silu(hnf[t] @ w1[e].float().T) * (hnf[t] @ w3[e].float().T)
            a = a.to(torch.bfloat16).float()  # the kernel stores the gated product in bf16
            ref[t] += float(o_w[t, s]) * (a @ w2[e].float().T)
    err = (xo.cpu() - ref).abs().max().item()
    assert err <= 1e-2 * max(1.0, ref.abs().max().item()), err


def test_rmsnorm_pack_and_embed(K):
    from oracle import bind as orc
    T, H, V = 5, 1024, 64
    g = torch.Generator().manual_seed(3)
    table_ = rand_bf16(V, H, gen=g).cuda()
    toks = torch.tensor([3, 0, 63, 7, 7], dtype=torch.int32, device="cuda")
    x = torch.zeros(T, H, device="cuda")
    K.embed(ptr(toks), ptr(table_), T, H, ptr(x), stream())
    gamma = rand_bf16(H, gen=g).cuda()
    R = 16
    out = torch.zeros(R * H, dtype=torch.int16, device="cuda")
    K.rmsnorm_pack(ptr(x), ptr(gamma), T, H, 1e-5, ptr(out), R, stream())
    torch.cuda.synchronize()
    assert torch.equal(x.cpu(), table_.cpu()[toks.cpu().long()].float())
    packed = out.cpu().numpy().view(np.uint16)
    rows = np.empty((T, H), np.uint16)
    K.unpack_rows(packed.ctypes.data_as(C.c_void_p), R, T, H, rows.ctypes.data_as(C.c_void_p))
    ref = orc.rmsnorm(x.cpu().numpy(), bf16_bits(gamma.cpu()), 1e-5, round_bf16=True)
    got = orc.bf16_to_f32(rows)
    assert np.abs(got - ref).max() <= 1e-2 * np.abs(ref).max()


@pytest.mark.parametrize("nq,nkv", [(8, 2), (12, 2), (16, 2), (2, 2)])
def test_rope_and_paged_attention(K, nq, nkv):
    """rope_qkv + kv_append + gqa_decode_paged against the fp32 oracle for
    G = n_q/n_kv in {4 (8x7B), 6 (8x22B/DBRX), 8, 1}; ragged contexts incl.
    1, page-1, page, page+1 tokens."""
    from oracle import bind as orc
    T, d, page = 6, 128, 16
    W = (nq + 2 * nkv) * d
    g = torch.Generator().manual_seed(5)
    ctx = np.array([1, 15, 16, 17, 100, 300], np.int32)
    pos = ctx - 1
    qkv = torch.randn(T, W, generator=g)
    rope = np.zeros((512, d // 2, 2), np.float32)
    K.rope_table(512, d, 1e6, rope.ctypes.data_as(C.c_void_p))
    rope_d = torch.from_numpy(rope).cuda()
    qkv_d, pos_d = qkv.cuda(), torch.from_numpy(pos).cuda()
    rb = torch.zeros(T, W, dtype=torch.int16, device="cuda")
    K.rope_qkv(ptr(qkv_d), ptr(pos_d), ptr(rope_d), T, nq, nkv, d, ptr(rb), stream())
    torch.cuda.synchronize()
    roped = orc.rope(qkv.numpy()[:, :(nq + nkv) * d], pos, nq + nkv, d, 1e6)
    got = orc.bf16_to_f32(rb.cpu().numpy().view(np.uint16))
    assert np.abs(got[:, :(nq + nkv) * d] - roped).max() < 2e-2
    assert np.abs(got[:, (nq + nkv) * d:] - qkv.numpy()[:, (nq + nkv) * d:]).max() < 2e-2

    # paged cache: random history for positions < pos, this step's k/v appended by the kernel
    cap = 320
    max_pages = cap // page
    n_pages = T * max_pages
    perm_pages = np.random.default_rng(0).permutation(n_pages).astype(np.int32)
    bt = perm_pages.reshape(T, max_pages)
    kpool = torch.zeros(n_pages * nkv * page * d, dtype=torch.int16, device="cuda")
    vpool = torch.zeros_like(kpool)
    hist_k = orc.f32_to_bf16(np.random.default_rng(1).uniform(-1, 1, (T, cap, nkv, d)))
    hist_v = orc.f32_to_bf16(np.random.default_rng(2).uniform(-1, 1, (T, cap, nkv, d)))
    kp = np.zeros((n_pages, nkv, page, d), np.uint16)
    vp = np.zeros_like(kp)
    # swizzled page rows (common.cuh kv_page_off): chunk c of token r at c ^ (r & 7)
    def swz(row, r):
        return row.reshape(nkv, d // 8, 8)[:, np.arange(d // 8) ^ (r & 7)].reshape(nkv, d)
    for t in range(T):
        for j in range(pos[t]):
            pid = bt[t, j // page]
            kp[pid, :, j % page] = swz(hist_k[t, j], j % page)
            vp[pid, :, j % page] = swz(hist_v[t, j], j % page)
    kpool.copy_(torch.from_numpy(kp.reshape(-1).view(np.int16)))
    vpool.copy_(torch.from_numpy(vp.reshape(-1).view(np.int16)))
    bt_d = torch.from_numpy(bt).cuda()
    seq = torch.arange(T, dtype=torch.int32, device="cuda")
    ctx_d = torch.from_numpy(ctx).cuda()
    K.kv_append(ptr(rb), nq, nkv, d, ptr(seq), ptr(pos_d), T, ptr(bt_d), max_pages, page,
                ptr(kpool), ptr(vpool), stream())
    out = torch.zeros(T, nq * d, device="cuda")
    R = 16
    outp = torch.zeros(R * nq * d, dtype=torch.int16, device="cuda")
    K.gqa_decode_paged(ptr(rb), W, ptr(kpool), ptr(vpool), ptr(bt_d), max_pages, ptr(seq),
                       ptr(ctx_d), T, nq, nkv, d, page, ptr(outp), R, ptr(out), stream())
    torch.cuda.synchronize()
    rbn = rb.cpu().numpy().view(np.uint16)
    for t in range(T):  # the appended step
        hist_k[t, pos[t]] = rbn[t, nq * d:(nq + nkv) * d].reshape(nkv, d)
        hist_v[t, pos[t]] = rbn[t, (nq + nkv) * d:].reshape(nkv, d)
    q = orc.bf16_to_f32(rbn[:, :nq * d])
    ref = orc.attention(q, hist_k, hist_v, ctx, nq, nkv, d)
    assert np.abs(out.cpu().numpy() - ref).max() < 2e-3
    # split-KV (flash-decoding over CTAs): splits > pages of the short
    # contexts included (empty splits), auto choice, and the counters must be
    # left at zero for the next launch
    scratch = torch.zeros(T * nq * 8 * 130, device="cuda")
    counters = torch.zeros(T * nkv, dtype=torch.int32, device="cuda")
    # stream-K decode over the flattened (token, head, page) space: the default
    # grid (2 CTAs per SM: more warps than pages here, so single-page ranges and
    # many-part merges) and small grids (multi-segment ranges)
    fscratch = torch.zeros(296 * 4 * 2 * (nq // nkv) * 130, device="cuda")
    fcount = torch.zeros(T * nkv, dtype=torch.int32, device="cuda")
    for ctas in (0, 1, 3, 7):
        out3 = torch.zeros_like(out)
        outp3 = torch.zeros_like(outp)
        K.gqa_decode_paged_flat(ptr(rb), W, ptr(kpool), ptr(vpool), ptr(bt_d), max_pages, ptr(seq), ptr(ctx_d), T,
                                nq, nkv, d, page, ptr(outp3), R, ptr(out3), ctas, ptr(fscratch), ptr(fcount), stream())
        torch.cuda.synchronize()
        assert np.abs(out3.cpu().numpy() - ref).max() < 2e-3, ctas
        assert int(fcount.abs().sum()) == 0
    for splits in (2, 3, 8, 0, 8):
        out2 = torch.zeros_like(out)
        outp2 = torch.zeros_like(outp)
        K.gqa_decode_paged_split(ptr(rb), W, ptr(kpool), ptr(vpool), ptr(bt_d), max_pages, ptr(seq),
                                 ptr(ctx_d), T, nq, nkv, d, page, ptr(outp2), R, ptr(out2), splits, 8,
                                 ptr(scratch), ptr(counters), stream())
        torch.cuda.synchronize()
        assert np.abs(out2.cpu().numpy() - ref).max() < 2e-3, splits
        assert int(counters.abs().sum()) == 0


def test_argmax(K):
    T, V = 3, 32000
    lg = torch.randn(T, V, device="cuda")
    lg[1, 17] = 100.0
    lg[1, 5] = 100.0  # tie -> lower index
    ids = torch.zeros(T, dtype=torch.int32, device="cuda")
    mg = torch.zeros(T, device="cuda")
    K.argmax(ptr(lg), T, V, ptr(ids), ptr(mg), stream())
    torch.cuda.synchronize()
    ref = lg.cpu().argmax(dim=1)
    assert ids[0].item() == ref[0].item() and ids[2].item() == ref[2].item()
    assert ids[1].item() == 5 and mg[1].item() == 0.0
    top2 = lg[0].topk(2).values
    assert abs(mg[0].item() - (top2[0] - top2[1]).item()) < 1e-6


def _tiles(lens):
    tiles, r = [], 0
    for n in lens:
        for q0 in range(0, n, 16):
            tiles.append((r, n, q0, 0))
        r += n
    return np.array(tiles, np.int32).reshape(-1)


@pytest.mark.parametrize("nq,nkv", [(8, 2), (12, 2), (4, 4), (8, 1)])
def test_prefill_attention_ragged_vs_fp32(K, nq, nkv):
    """Causal GQA prefill attention (attention_prefill.cu) on ragged
    sequences vs a torch fp32 reference on the same bf16 inputs."""
    from oracle import bind as orc
    d = 128
    lens = [1, 17, 64, 100, 33, 16, 130]
    T, W = sum(lens), (nq + 2 * nkv) * d
    g = torch.Generator().manual_seed(7)
    qkv = (torch.rand(T, W, generator=g) * 2 - 1).to(torch.bfloat16)
    qkv_d = qkv.cuda()
    tiles = torch.from_numpy(_tiles(lens)).cuda()
    R = (T + 15) // 16 * 16
    outp = torch.zeros(R * nq * d, dtype=torch.int16, device="cuda")
    K.prefill_attention(ptr(qkv_d), W, ptr(tiles), tiles.numel() // 4, nq, nkv, d, ptr(outp), R, stream())
    torch.cuda.synchronize()
    packed = outp.cpu().numpy().view(np.uint8)
    rows = np.zeros((T, nq * d), np.uint16)
    K.unpack_rows(packed.ctypes.data_as(C.c_void_p), R, T, nq * d, rows.ctypes.data_as(C.c_void_p))
    got = orc.bf16_to_f32(rows)
    x = qkv.float()
    ref = np.zeros((T, nq * d), np.float32)
    r = 0
    G = nq // nkv
    for n in lens:
        q = x[r:r + n, :nq * d].reshape(n, nq, d)
        k = x[r:r + n, nq * d:(nq + nkv) * d].reshape(n, nkv, d)
        v = x[r:r + n, (nq + nkv) * d:].reshape(n, nkv, d)
        kk = k.repeat_interleave(G, dim=1)
        vv = v.repeat_interleave(G, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, kk) / np.sqrt(d)
        mask = torch.triu(torch.ones(n, n, dtype=torch.bool), 1)
        s = s.masked_fill(mask, float("-inf"))
        o = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), vv)
        ref[r:r + n] = o.reshape(n, nq * d).numpy()
        r += n
    err = np.abs(got - ref)
    assert err.max() < 1.5e-2, err.max()
    assert err.mean() < 2e-3, err.mean()


def test_kv_stage_layout(K):
    nq, nkv, d = 8, 2, 128
    lens = [3, 17, 1, 40]
    T, W = sum(lens), (nq + 2 * nkv) * d
    qkv = torch.randint(-30000, 30000, (T, W), dtype=torch.int16, device="cuda")
    tok_seq = np.concatenate([np.full(n, j, np.int32) for j, n in enumerate(lens)])
    tok_pos = np.concatenate([np.arange(n, dtype=np.int32) for n in lens])
    row0 = np.cumsum([0] + lens[:-1]).astype(np.int32)
    ts, tp, r0, ln = (torch.from_numpy(a).cuda() for a in (tok_seq, tok_pos, row0, np.array(lens, np.int32)))
    sk = torch.zeros(T * nkv * d, dtype=torch.int16, device="cuda")
    sv = torch.zeros_like(sk)
    K.kv_stage(ptr(qkv), W, nq, nkv, d, ptr(ts), ptr(tp), ptr(r0), ptr(ln), T, ptr(sk), ptr(sv), stream())
    torch.cuda.synchronize()
    q = qkv.cpu().numpy()
    for j, n in enumerate(lens):
        seg_k = sk.cpu().numpy()[row0[j] * nkv * d:(row0[j] + n) * nkv * d].reshape(nkv, n, d)
        seg_v = sv.cpu().numpy()[row0[j] * nkv * d:(row0[j] + n) * nkv * d].reshape(nkv, n, d)
        rows = q[row0[j]:row0[j] + n]
        assert np.array_equal(seg_k, rows[:, nq * d:(nq + nkv) * d].reshape(n, nkv, d).transpose(1, 0, 2))
        assert np.array_equal(seg_v, rows[:, (nq + nkv) * d:].reshape(n, nkv, d).transpose(1, 0, 2))


def encode_weight_dev(K, w_bf16, fmt=1):
    """Host-pack + codec-encode a [M, K] bf16 weight and upload; returns (device
    buffer, encoded row-block pointers).  fmt 3: the row-plane code of the
    TMEM-operand engine (see encode_rows_dev)."""
    if fmt in (3, 4):
        dev, blocks, flags = encode_rows_dev(K, w_bf16, fmt=fmt)
        assert not any(flags)  # encoded-size ring slots (codec_raw = 0)
        return dev, blocks
    M, Kd = w_bf16.shape
    src = bf16_bits(w_bf16.cpu())
    packed = np.empty_like(src)
    K.pack_weight(src.ctypes.data_as(C.c_void_p), M, Kd, packed.ctypes.data_as(C.c_void_p))
    enc = np.zeros(M // 128 * (Kd // 64) * 12432, np.uint8)
    K.codec_encode(packed.ctypes.data_as(C.c_void_p), M, Kd, enc.ctypes.data_as(C.c_void_p))
    dev = torch.from_numpy(enc).cuda()
    blocks = [dev.data_ptr() + rb * (Kd // 64) * 12432 for rb in range(M // 128)]
    return dev, blocks


def encode_rows_dev(K, w_bf16, force_raw=(), fmt=3, cap=44):
    """Codec-3 weight blocks (row-plane encoded tiles, mlt_codec_encode_rows),
    or with fmt 4 the 3-bit code (mlt_codec4_encode_rows, 11600 B tiles):
    a row block the code cannot hold (too many escapes in a tile), or listed in
    force_raw, is stored as raw packed tiles with its pointer tagged (bit 0).
    Returns (device buffer, row-block pointers, raw flags)."""
    if fmt == 4:
        tb = K.codec4_tile_bytes_for(cap)
        enc_fn = lambda src, m, k, dst, rr: K.codec4_encode_rows_cap(src, m, k, cap, dst, rr)  # noqa: E731
    else:
        enc_fn, tb = K.codec_encode_rows, 12432
    M, Kd = w_bf16.shape
    src = bf16_bits(w_bf16.cpu())
    packed = np.empty_like(src)
    K.pack_weight(src.ctypes.data_as(C.c_void_p), M, Kd, packed.ctypes.data_as(C.c_void_p))
    kb, rbs = Kd // 64, M // 128
    pb = packed.view(np.uint8).reshape(rbs, kb * 16384)
    parts, rel, flags = [], [], []
    off = 0
    for r in range(rbs):
        blk = np.empty(kb * 16384, np.uint8)
        rr = np.zeros(1, np.uint8)
        assert enc_fn(np.ascontiguousarray(pb[r]).ctypes.data_as(C.c_void_p), 128, Kd,
                      blk.ctypes.data_as(C.c_void_p), rr.ctypes.data_as(C.c_void_p)) >= 0
        raw = bool(rr[0]) or r in force_raw
        blk = pb[r].copy() if raw else blk[:kb * tb]
        parts.append(blk)
        rel.append((off, raw))
        flags.append(raw)
        off += blk.size
    dev = torch.from_numpy(np.concatenate(parts)).cuda()
    return dev, [dev.data_ptr() + o + (1 if raw else 0) for o, raw in rel], flags


@pytest.mark.parametrize("codec", [1, 3, 4])
@pytest.mark.parametrize("T,M,Kd,n_cap,splits,resid", [(16, 256, 512, 16, 1, True), (64, 384, 4096, 64, 3, False),
                                                        (256, 256, 1024, 256, 2, False),
                                                        (200, 128, 256, 208, 1, True)])
def test_codec_gemm_bitwise_equals_raw(K, T, M, Kd, n_cap, splits, resid, codec):
    """The GEMM on encoded weights (decoder warps expand tiles in smem) returns
    the same bits as on raw bf16 tiles: dense fp32 epilogue, split-K, residual."""
    g = torch.Generator().manual_seed(T + M + Kd)
    w = (unif_bf16 if codec == 4 else rand_bf16)(M, Kd, scale=Kd ** -0.5, gen=g)
    x = rand_bf16(T, Kd, gen=g)
    R = (T + 15) // 16 * 16
    raw_dev, raw_blocks = pack_weight_dev(K, w)  # keep the buffers alive while the GEMMs read them
    enc_dev, enc_blocks = encode_weight_dev(K, w, codec)
    xp = pack_rows_dev(K, x, R)
    res = torch.randn(T, M, device="cuda") if resid else None
    outs = []
    for cdc, blocks in ((0, raw_blocks), (codec, enc_blocks)):
        tab = table([blocks])
        out = torch.zeros(splits, R, M, device="cuda")
        a = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=1, RB=M // 128, K=Kd, b=xp.data_ptr(), R=R,
                          rows_dense=T, n_cap=n_cap, epi=0, alpha=1.0, out_f32=out.data_ptr(), ldo=M,
                          residual=res.data_ptr() if resid else None, ldr=M, k_splits=splits,
                          split_stride=R * M, codec=cdc)
        K.gemm(C.byref(a), stream())
        torch.cuda.synchronize()
        outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1])
    ref = x.float() @ w.float().T + (res.cpu() if resid else 0)
    assert (outs[1].sum(0)[:T] - ref).abs().max().item() <= 2e-3 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("codec", [1, 3, 4])
@pytest.mark.parametrize("T,H,Fd,E,Kk,n_cap", [(64, 512, 768, 8, 2, 64), (33, 256, 256, 16, 4, 32)])
def test_codec_expert_ffn_bitwise_equals_raw(K, T, H, Fd, E, Kk, n_cap, codec):
    """Grouped gate/up (two encoded matrices, fused SiLU -> packed bf16) and
    down on encoded experts == the raw-tile GEMMs, bit for bit."""
    hn, w1, w3, w2, wr = _expert_setup(T, H, Fd, E, Kk, seed=T + H + 1, uniform=codec == 4)
    hn_d, wr_d = hn.cuda(), wr.cuda()
    idx = torch.zeros(T, Kk, dtype=torch.int32, device="cuda")
    wts = torch.zeros(T, Kk, device="cuda")
    K.router_topk(None, None, 0.0, ptr(hn_d), ptr(wr_d), T, H, E, Kk, None, None, ptr(idx), ptr(wts), stream())
    R = (T * Kk + 16 * E + 15) // 16 * 16
    cnt = torch.zeros(E, dtype=torch.int32, device="cuda")
    off = torch.zeros(E + 1, dtype=torch.int32, device="cuda")
    perm = torch.zeros(R, dtype=torch.int32, device="cuda")
    inv = torch.zeros(T * Kk, dtype=torch.int32, device="cuda")
    xp = torch.zeros(R * H, dtype=torch.int16, device="cuda")
    K.moe_permute(ptr(idx), ptr(hn_d), T, H, E, Kk, ptr(cnt), ptr(off), ptr(perm), ptr(inv), ptr(xp), R, stream())
    results = []
    keep = []
    for cdc in (0, codec):
        mk = (lambda K_, w_: encode_weight_dev(K_, w_, cdc)) if cdc else pack_weight_dev
        t13, t2 = [], []
        for m in (w1, w3):
            for w in m:
                dev, bl = mk(K, w)
                keep.append(dev)
                t13.append(bl)
        for w in w2:
            dev, bl = mk(K, w)
            keep.append(dev)
            t2.append(bl)
        tab13, tab2 = table(t13), table(t2)
        inter = torch.zeros(R * Fd, dtype=torch.int16, device="cuda")
        y = torch.zeros(R, H, device="cuda")
        gu = capi.GemmArgs(a_table=tab13.data_ptr(), n_mats=2, G=E, RB=Fd // 128, K=H, b=xp.data_ptr(), R=R,
                           b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=n_cap, epi=1, alpha=1.0,
                           out_packed=inter.data_ptr(), out_R=R, codec=cdc)
        K.gemm(C.byref(gu), stream())
        dn = capi.GemmArgs(a_table=tab2.data_ptr(), n_mats=1, G=E, RB=H // 128, K=Fd, b=inter.data_ptr(), R=R,
                           b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=n_cap, epi=0, alpha=1.0,
                           out_f32=y.data_ptr(), ldo=H, codec=cdc)
        K.gemm(C.byref(dn), stream())
        torch.cuda.synchronize()
        results.append((inter.cpu(), y.cpu()))
    assert torch.equal(results[0][0], results[1][0])
    assert torch.equal(results[0][1], results[1][1])



@pytest.mark.parametrize("codec", [3, 4])
@pytest.mark.parametrize("T,M,Kd,n_cap,splits", [(16, 512, 1024, 16, 1), (80, 384, 2048, 96, 2)])
def test_codec3_escapes_and_raw_blocks(K, T, M, Kd, n_cap, splits, codec):
    """Codec 3 (row-plane tiles decoded into TMEM, MMA with A from TMEM) on
    heavy-tailed weights: tiles with escapes (patched per row in registers),
    row blocks the code cannot hold stored raw (tagged pointers), plus a
    forced raw block — bit-equal to the raw-tile GEMM."""
    g = torch.Generator().manual_seed(M + Kd + 3)
    w = (unif_bf16 if codec == 4 else rand_bf16)(M, Kd, scale=Kd ** -0.5, gen=g)
    # sparse outliers: a few per tile in rows 0..127 -> escapes; a wide
    # spread in the last row block -> more than 31 escapes -> raw
    nout = M * Kd // 2048
    ri = torch.randint(0, M - 128, (nout,), generator=g)
    ci = torch.randint(0, Kd, (nout,), generator=g)
    w[ri, ci] = (torch.rand(nout, generator=g) * 64 + 1).to(torch.bfloat16)
    w[M - 128:] = (torch.randn(128, Kd, generator=g) * torch.exp(torch.randn(128, Kd, generator=g) * 4)).to(torch.bfloat16)
    x = rand_bf16(T, Kd, gen=g)
    R = (T + 15) // 16 * 16
    raw_dev, raw_blocks = pack_weight_dev(K, w)
    enc_dev, enc_blocks, flags = encode_rows_dev(K, w, force_raw=(1,), fmt=codec)
    assert flags[-1] and flags[1] and not flags[0], flags
    xp = pack_rows_dev(K, x, R)
    outs = []
    for cdc, blocks in ((0, raw_blocks), (codec, enc_blocks)):
        tab = table([blocks])
        out = torch.zeros(splits, R, M, device="cuda")
        a = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=1, RB=M // 128, K=Kd, b=xp.data_ptr(), R=R,
                          rows_dense=T, n_cap=n_cap, epi=0, alpha=1.0, out_f32=out.data_ptr(), ldo=M,
                          k_splits=splits, split_stride=R * M, codec=cdc, codec_raw=int(cdc != 0))
        K.gemm(C.byref(a), stream())
        torch.cuda.synchronize()
        outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("T,n_cap", [(48, 48), (130, 144)])
def test_codec4_phase_override_escapes(K, T, n_cap):
    """Codec 4 tiles of every kind the encoder emits: phase 0 and phase 1
    tiles (top binade alone in its high-byte pair), rows whose out-of-table
    weights go through the row's slot-7 override, escapes in every row quarter
    up to the 48-entry cap, a raw block — the TMEM-operand GEMM equals the
    raw-tile GEMM bit for bit."""
    g = torch.Generator().manual_seed(T + 17)
    M, Kd = 512, 512
    a = 1.5 * 2.0 ** -7
    w = ((torch.rand(M, Kd, generator=g) * 2 - 1) * a)
    w[128:256] *= 2                        # the other binade alignment (phase 0)
    w[256:384, :8] = 2.0 ** -30            # rows with one repeated tiny value: slot-7 overrides
    # tiles with many escapes: distinct tiny values spread over rows of every quarter
    idx = torch.randperm(128 * Kd, generator=g)[:26 * (Kd // 64)]
    vals = torch.pow(2.0, -torch.randint(20, 60, (idx.numel(),), generator=g).float())
    w[:128].view(-1)[idx] = vals * torch.sign(torch.rand(idx.numel(), generator=g) - 0.5)
    w = w.to(torch.bfloat16)
    x = rand_bf16(T, Kd, gen=g)
    R = (T + 15) // 16 * 16
    raw_dev, raw_blocks = pack_weight_dev(K, w)
    enc_dev, enc_blocks, flags = encode_rows_dev(K, w, force_raw=(3,), fmt=4)
    assert flags == [False, False, False, True], flags
    xp = pack_rows_dev(K, x, R)
    outs = []
    for cdc, blocks in ((0, raw_blocks), (4, enc_blocks)):
        tab = table([blocks])
        out = torch.zeros(1, R, M, device="cuda")
        args = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=1, RB=M // 128, K=Kd, b=xp.data_ptr(), R=R,
                             rows_dense=T, n_cap=n_cap, epi=0, alpha=1.0, out_f32=out.data_ptr(), ldo=M,
                             k_splits=1, split_stride=R * M, codec=cdc, codec_raw=int(cdc != 0))
        K.gemm(C.byref(args), stream())
        torch.cuda.synchronize()
        outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("cap", [0, 80, 200])
def test_codec4_tile_capacity(K, cap):
    """Codec 4 tiles of a non-default capacity (GemmArgs enc_tile = 11424 +
    4 cap bytes, the runtime's per-weight-kind sizing): DBRX-down-scale
    weights (1.07 * 2^-6, ~31 entries per tile) at cap 80 and 200 code every
    block; cap 0 (no records or escapes) leaves only blocks without them,
    the rest raw — all bit-equal to the raw-tile GEMM."""
    g = torch.Generator().manual_seed(cap + 5)
    M, Kd, T = 384, 1024, 40
    w = unif_bf16(M, Kd, scale=10752 ** -0.5, gen=g)
    x = rand_bf16(T, Kd, gen=g)
    R = (T + 15) // 16 * 16
    raw_dev, raw_blocks = pack_weight_dev(K, w)
    enc_dev, enc_blocks, flags = encode_rows_dev(K, w, fmt=4, cap=cap)
    assert (not any(flags)) if cap else all(flags)
    xp = pack_rows_dev(K, x, R)
    outs = []
    for cdc, blocks in ((0, raw_blocks), (4, enc_blocks)):
        tab = table([blocks])
        out = torch.zeros(1, R, M, device="cuda")
        args = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=1, RB=M // 128, K=Kd, b=xp.data_ptr(), R=R,
                             rows_dense=T, n_cap=48, epi=0, alpha=1.0, out_f32=out.data_ptr(), ldo=M,
                             k_splits=1, split_stride=R * M, codec=cdc, codec_raw=int(any(flags)),
                             enc_tile=K.codec4_tile_bytes_for(cap) if cdc else 0)
        K.gemm(C.byref(args), stream())
        torch.cuda.synchronize()
        outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1])


def encode_frag_dev(K, w_bf16, raw_rows=()):
    """Codec-2 weight blocks (fragment-order encoded tiles, gemm_codec.cu):
    row blocks listed in raw_rows are stored as raw fragment-order tiles with
    their page-table pointer tagged (bit 0), the runtime's per-block fallback.
    Returns (device buffer, row-block pointers)."""
    M, Kd = w_bf16.shape
    src = bf16_bits(w_bf16.cpu())
    packed = np.empty_like(src)
    K.pack_weight(src.ctypes.data_as(C.c_void_p), M, Kd, packed.ctypes.data_as(C.c_void_p))
    kb, rbs = Kd // 64, M // 128
    pb = packed.view(np.uint8).reshape(rbs, kb * 16384)
    parts, ptrs_rel = [], []
    off = 0
    for r in range(rbs):
        if r in raw_rows:
            blk = np.empty(kb * 16384, np.uint8)
            K.frag_pack(pb[r].ctypes.data_as(C.c_void_p), kb, blk.ctypes.data_as(C.c_void_p))
        else:
            blk = np.empty(kb * 12432, np.uint8)
            rr = np.zeros(1, np.uint8)
            assert K.codec_encode_frag(np.ascontiguousarray(pb[r]).ctypes.data_as(C.c_void_p), 128, Kd,
                                       blk.ctypes.data_as(C.c_void_p), rr.ctypes.data_as(C.c_void_p)) == 0
        parts.append(blk)
        ptrs_rel.append((off, r in raw_rows))
        off += blk.size
        off = (off + 15) // 16 * 16
        parts.append(np.zeros((-blk.size) % 16, np.uint8))
    dev = torch.from_numpy(np.concatenate(parts)).cuda()
    return dev, [dev.data_ptr() + o + (1 if raw else 0) for o, raw in ptrs_rel]


@pytest.mark.parametrize("T,M,Kd,n_cap,splits,resid", [(16, 256, 512, 16, 1, True), (64, 384, 4096, 64, 3, False),
                                                        (37, 256, 1024, 48, 2, False), (100, 128, 256, 64, 1, True)])
def test_codec2_gemm_register_decode(K, T, M, Kd, n_cap, splits, resid):
    """Register-decode GEMM (codec = 2: fragment-order encoded tiles, mma.sync):
    against torch fp32; and encoded == raw fallback blocks (tagged pointers,
    same kernel without the decode) bit for bit, for all-raw and mixed tables —
    the GPU decode is exact.  Token counts above n_cap loop over chunks."""
    g = torch.Generator().manual_seed(T + M + Kd + 7)
    w = rand_bf16(M, Kd, scale=Kd ** -0.5, gen=g)
    x = rand_bf16(T, Kd, gen=g)
    R = (T + 15) // 16 * 16
    xp = pack_rows_dev(K, x, R)
    res = torch.randn(T, M, device="cuda") if resid else None
    outs = []
    for raw_rows in ((), tuple(range(M // 128)), (0,)):
        dev, blocks = encode_frag_dev(K, w, raw_rows)
        tab = table([blocks])
        out = torch.zeros(splits, R, M, device="cuda")
        a = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=1, RB=M // 128, K=Kd, b=xp.data_ptr(), R=R,
                          rows_dense=T, n_cap=n_cap, epi=0, alpha=1.0, out_f32=out.data_ptr(), ldo=M,
                          residual=res.data_ptr() if resid else None, ldr=M, k_splits=splits,
                          split_stride=R * M, codec=2, codec_raw=int(bool(raw_rows)))
        K.gemm(C.byref(a), stream())
        torch.cuda.synchronize()
        outs.append(out.cpu())
        del dev
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    ref = x.float() @ w.float().T + (res.cpu() if resid else 0)
    assert (outs[0].sum(0)[:T] - ref).abs().max().item() <= 2e-3 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("T,H,Fd,E,Kk", [(64, 512, 768, 8, 2), (33, 256, 256, 16, 4), (96, 256, 512, 2, 1)])
def test_codec2_expert_ffn_register_decode(K, T, H, Fd, E, Kk):
    """Grouped gate/up (fused SiLU -> packed bf16, <= 32 tokens per chunk) and
    down (<= 64 tokens per chunk, 2 K-splits) on codec-2 experts: against a
    torch fp32 reference of the same routing, and bit-equal to raw fallback
    blocks (E = 2, top-1 puts > 32 tokens on an expert: chunk loop)."""
    hn, w1, w3, w2, wr = _expert_setup(T, H, Fd, E, Kk, seed=T + H + 5)
    hn_d, wr_d = hn.cuda(), wr.cuda()
    idx = torch.zeros(T, Kk, dtype=torch.int32, device="cuda")
    wts = torch.zeros(T, Kk, device="cuda")
    K.router_topk(None, None, 0.0, ptr(hn_d), ptr(wr_d), T, H, E, Kk, None, None, ptr(idx), ptr(wts), stream())
    R = (T * Kk + 16 * E + 15) // 16 * 16
    cnt = torch.zeros(E, dtype=torch.int32, device="cuda")
    off = torch.zeros(E + 1, dtype=torch.int32, device="cuda")
    perm = torch.zeros(R, dtype=torch.int32, device="cuda")
    inv = torch.zeros(T * Kk, dtype=torch.int32, device="cuda")
    xp = torch.zeros(R * H, dtype=torch.int16, device="cuda")
    K.moe_permute(ptr(idx), ptr(hn_d), T, H, E, Kk, ptr(cnt), ptr(off), ptr(perm), ptr(inv), ptr(xp), R, stream())
    results = []
    for all_raw in (False, True):
        keep, t13, t2 = [], [], []
        for m in (w1, w3):
            for w in m:
                dev, bl = encode_frag_dev(K, w, tuple(range(w.shape[0] // 128)) if all_raw else ())
                keep.append(dev)
                t13.append(bl)
        for w in w2:
            dev, bl = encode_frag_dev(K, w, tuple(range(w.shape[0] // 128)) if all_raw else ())
            keep.append(dev)
            t2.append(bl)
        tab13, tab2 = table(t13), table(t2)
        inter = torch.zeros(R * Fd, dtype=torch.int16, device="cuda")
        y = torch.zeros(2, R, H, device="cuda")
        gu = capi.GemmArgs(a_table=tab13.data_ptr(), n_mats=2, G=E, RB=Fd // 128, K=H, b=xp.data_ptr(), R=R,
                           b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=32, epi=1, alpha=1.0,
                           out_packed=inter.data_ptr(), out_R=R, codec=2, codec_raw=int(all_raw))
        K.gemm(C.byref(gu), stream())
        dn = capi.GemmArgs(a_table=tab2.data_ptr(), n_mats=1, G=E, RB=H // 128, K=Fd, b=inter.data_ptr(), R=R,
                           b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=64, epi=0, alpha=1.0,
                           out_f32=y.data_ptr(), ldo=H, codec=2, k_splits=2, split_stride=R * H,
                           codec_raw=int(all_raw))
        K.gemm(C.byref(dn), stream())
        torch.cuda.synchronize()
        results.append((inter.cpu(), y.cpu()))
    assert torch.equal(results[0][0], results[1][0]) and torch.equal(results[0][1], results[1][1])
    # torch fp32 reference of every (token, slot) row
    inter_rows = np.empty((R, Fd), np.uint16)
    K.unpack_rows(results[0][0].numpy().ctypes.data_as(C.c_void_p), R, R, Fd, inter_rows.ctypes.data_as(C.c_void_p))
    cnt_h, off_h, perm_h = cnt.cpu().numpy(), off.cpu().numpy(), perm.cpu().numpy()
    yh = results[0][1].sum(0)
    hnf = hn.float()
    worst_i = worst_y = 0.0
    for e in range(E):
        for r in range(int(cnt_h[e])):
            row = int(off_h[e]) + r
            t = int(perm_h[row]) // Kk
            g_ = hnf[t] @ w1[e].float().T
            u_ = hnf[t] @ w3[e].float().T
            it = torch.nn.functional.silu(g_) * u_
            got_i = torch.from_numpy(inter_rows[row].astype(np.int32) << 16).view(torch.float32)
            worst_i = max(worst_i, ((got_i - it).abs().max() / it.abs().max()).item())
            yr = got_i.to(torch.bfloat16).float() @ w2[e].float().T
            worst_y = max(worst_y, ((yh[row] - yr).abs().max() / yr.abs().max()).item())
    assert worst_i < 1.5e-2 and worst_y < 2e-3, (worst_i, worst_y)

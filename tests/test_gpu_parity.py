"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical seeded
inputs.  Bars:
  * plan / mask / block-list / interval / work-list outputs: bit-exact;
  * keep-count increments: bit-exact against the oracle's selection run on the GPU's own fp32 E;
  * E: |dE| <= 5e-5 (fp32 exp2 path vs fp64), row sums 1 +- 1e-4;
  * attention (bf16 I/O, fp32 accumulation): max |dO| <= 2e-2, mean |dO| <= 2e-3 (north star);
    lse |d| <= 1e-3.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_05503_b200 import inputs
from paper_2603_05503_b200.inputs import CONFIGS, Layout, qkv

pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


@pytest.fixture(scope="module")
def csa():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2603_05503_b200 import _build

    _build.build()
    from paper_2603_05503_b200 import csa as m

    return m


def head64(t, b, h):
    return t[b, :, h].double().cpu().numpy()


def u16_zeros(n):
    return torch.zeros(n, dtype=torch.int16, device="cuda").view(torch.uint16)


def u16_np(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def u16_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint16).reshape(-1).view(np.int16)).cuda().view(torch.uint16)


def unpack_bits(words, nb):
    w = words.view(np.uint32) if words.dtype != np.uint32 else words
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")
    return bits.reshape(-1, ((nb + 31) // 32) * 32)[:, :nb]


def check_plan_against_oracle(csa, lay, counts_np, min_count, sim=None, gamma=0.87, anchor_k=5):
    dev = torch.device("cuda")
    cells = counts_np.shape[0]
    counts = u16_dev(counts_np)
    simt = None if sim is None else torch.tensor(sim, dtype=torch.float64, device=dev)
    plan = csa.compile_plan(lay, counts, min_count, similarity=simt, gamma=gamma, anchor_k=anchor_k)
    csa.validate_plan(plan)
    nb, nbk = lay.NB, lay.NBK
    kind = plan.kind.cpu().numpy()
    bits = unpack_bits(plan.mask_bits.cpu().numpy(), nbk).reshape(cells, nb, nbk)
    brp = plan.blk_row_ptr.cpu().numpy().reshape(cells, nb + 1)
    irp = plan.ivl_row_ptr.cpu().numpy().reshape(cells, nb + 1)
    bb = plan.blk_base.cpu().numpy()
    ib = plan.ivl_base.cpu().numpy()
    bidx = u16_np(plan.blk_idx)
    ivl = u16_np(plan.ivl)
    area = plan.kept_area.cpu().numpy()
    for c in range(cells):
        ref = oracle.compile_cell(counts_np[c], lay.N, lay.B, lay.F, lay.H, lay.W, min_count,
                                  similarity=None if sim is None else sim[c], gamma=gamma,
                                  anchor_k=anchor_k, block_kv=lay.BK or None)
        assert kind[c] == ref["kind"]
        assert area[c] == ref["kept_area"]
        assert np.array_equal(brp[c], ref["blk_row_ptr"])
        assert np.array_equal(irp[c], ref["ivl_row_ptr"])
        if ref["kind"] == 0:
            assert np.array_equal(bits[c], ref["mask"])
            assert np.array_equal(bidx[bb[c]:bb[c + 1]], ref["blk_idx"])
            assert np.array_equal(ivl[2 * ib[c]:2 * ib[c + 1]].reshape(-1, 2), ref["ivl"])
        else:
            assert not bits[c].any() and bb[c + 1] == bb[c]
    return plan


# ---------------------------------------------------------------- a6 plan compiler
@pytest.mark.parametrize("lay", [Layout(2, 5, 25, 64), Layout(4, 8, 8, 64), Layout(21, 30, 52, 128),
                                 Layout(3, 7, 100, 128)])
def test_plan_compile_bit_exact(csa, lay):
    nb = lay.NB
    counts = inputs.random_counts(nb, 5, 64, seed=nb)
    counts[1] = 0                                   # every row repaired -> argmax (c = 0)
    counts[2] = 64                                  # all ones
    counts[3] = 0
    counts[3][:, ::2] = 40                          # alternating: worst-case intervals
    check_plan_against_oracle(csa, lay, counts, 32)
    sim = [0.5, 0.87, 0.8700001, 1.0, 0.0]          # s == gamma stays MASK (strict, Q8)
    check_plan_against_oracle(csa, lay, counts, 32, sim=sim, anchor_k=min(5, lay.H))


@pytest.mark.parametrize("field,value", [("kind", 2), ("anchor_k", 0), ("anchor_k", 99),
                                         ("blk_base", -1), ("blk_row_ptr", 5), ("ivl_row_ptr", 3)])
def test_validate_rejects_corrupt_plan_fields(csa, field, value):
    """csa_validate_plan flags out-of-range kinds / anchor counts and bases or row pointers that
    do not start at 0 (a CRC-valid file with anchor_k = 0 used to pass)."""
    lay = Layout(2, 9, 40, 128)
    rng = np.random.default_rng(2)
    counts = u16_dev((rng.random((2, lay.NB, lay.NB)) < 0.5).astype(np.uint16))
    sim = torch.tensor([0.0, 1.0], dtype=torch.float64, device="cuda")
    plan = csa.compile_plan(lay, counts, 1, similarity=sim, gamma=0.87, anchor_k=3)
    csa.validate_plan(plan)
    t = getattr(plan, field)
    idx = 1 if field in ("kind", "anchor_k") else 0   # cell 1 is REPETITIVE
    t[idx] = value
    with pytest.raises(csa.CsaError, match="CORRUPT_PLAN"):
        csa.validate_plan(plan)


def test_plan_compile_wan720_synthetic(csa):
    cfg = CONFIGS["wan720"]
    counts = inputs.synthetic_counts(cfg.layout, 4, cfg.sparsity, 64, seed=3)
    check_plan_against_oracle(csa, cfg.layout, counts, 32)


def test_work_list_bit_exact(csa):
    lay = Layout(21, 30, 52, 128)
    counts = inputs.random_counts(lay.NB, 6, 8, seed=5)
    sim = [0.0, 0.95, 0.0, 0.0, 0.99, 0.0]
    plan = check_plan_against_oracle(csa, lay, counts, 4, sim=sim, anchor_k=5)
    rp = plan.blk_row_ptr.cpu().numpy().reshape(6, lay.NB + 1)
    nnz = np.diff(rp, axis=1)
    kinds = plan.kind.cpu().numpy()
    ak = plan.anchor_k.cpu().numpy()
    for base, nh in ((0, 6), (1, 4)):
        wl = csa.build_work_list(plan, base, nh, order=0)
        got = wl.items.cpu().numpy().view(np.uint32)[: int(wl.n_work.item())]
        ref = oracle.work_list(lay.N, lay.B, lay.F, lay.W, kinds[base:base + nh], ak[base:base + nh],
                               nnz[base:base + nh])
        assert np.array_equal(got, ref)
        for order in (1, 2, 3):
            wl = csa.build_work_list(plan, base, nh, order=order)
            got = wl.items.cpu().numpy().view(np.uint32)[: int(wl.n_work.item())]
            ref = oracle.work_list(lay.N, lay.B, lay.F, lay.W, kinds[base:base + nh],
                                   ak[base:base + nh], nnz[base:base + nh], order=order)
            assert np.array_equal(got, ref), order


# ---------------------------------------------------------------- a7/a8 attention
def run_attention(csa, lay, q, k, v, masks=None, rep=None, anchor_k=2, order=2, lse=False):
    """masks: [H, NB, NBK] uint8 for MASK heads; rep: list of REPETITIVE head indices."""
    heads = q.shape[2]
    if masks is None:
        masks = np.ones((heads, lay.NB, lay.NBK), np.uint8)
    counts = masks.astype(np.uint16)
    sim = None
    if rep:
        sim = torch.tensor([1.0 if h in rep else 0.0 for h in range(heads)], dtype=torch.float64,
                           device="cuda")
    ct = u16_dev(counts)
    plan = csa.compile_plan(lay, ct, 1, similarity=sim, gamma=0.87, anchor_k=anchor_k)
    work = csa.build_work_list(plan, 0, heads, order=order)
    lse_t = torch.empty(q.shape[0] * heads * lay.N, dtype=torch.float32, device="cuda") if lse else None
    out = csa.sparse_attn_fwd(q, k, v, plan, work, lse_out=lse_t)
    torch.cuda.synchronize()
    return out, lse_t, plan


def fallback_count(csa, q):
    """Items the fixed-reference kernel (attn5.cu / attn_rect.cu) handed to the exact-max fallback
    passes in the last launch on q's device: uint32 at byte 256 of the attention workspace."""
    ws = csa._sched_workspace(q.device, 0)  # current stream: the one the test launched on
    return int(ws[256:260].view(torch.int32).item())


def oracle_head(lay, q, k, v, b, h, mask=None, rep_k=None, rows=None):
    scale = 1.0 / np.sqrt(q.shape[3])
    qh, kh, vh = head64(q, b, h), head64(k, b, h), head64(v, b, h)
    if rep_k:
        return oracle.anchor_attention_rows(lay.F, lay.H, lay.W, qh, kh, vh, scale, rep_k, rows)
    return oracle.masked_attention_rows(qh, kh, vh, scale, lay.B, mask, rows,
                                        block_kv=lay.BK or None)


def assert_close(got, ref, what=""):
    err = np.abs(got - ref)
    assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, f"{what} max {err.max()} mean {err.mean()}"


@pytest.mark.parametrize("name", ["tiny", "tiny_ragged"])
def test_attention_tiny_masks(csa, name):
    cfg = CONFIGS[name]
    lay = cfg.layout
    q, k, v = qkv(1, lay.N, 1, cfg.d, seed=0, device="cuda")
    nb = lay.NB
    cases = {"hand": inputs.TINY_HAND_MASK, "ones": np.ones((nb, nb), np.uint8),
             "identity": np.eye(nb, dtype=np.uint8),
             "last_col": np.eye(nb, dtype=np.uint8)[[nb - 1] * nb]}
    for cname, m in cases.items():
        out, lse, _ = run_attention(csa, lay, q, k, v, masks=m[None], lse=True)
        ref, ref_lse = oracle_head(lay, q, k, v, 0, 0, mask=m)
        assert_close(out[0, :, 0].double().cpu().numpy(), ref, cname)
        assert np.abs(lse.cpu().numpy() - ref_lse).max() <= 1e-3, cname


@pytest.mark.parametrize("lay,d", [(Layout(2, 9, 40, 128), 128), (Layout(2, 9, 40, 128), 64),
                                   (Layout(2, 5, 25, 64), 64)])
@pytest.mark.parametrize("jump", [3.0, 40.0])
def test_attention_running_max_jumps(csa, lay, d, jump):
    """Key blocks whose scores grow block by block: later tiles exceed the first tile's max (the
    fixed reference of the block-128 kernels; the running max and lazy rescale of attn.cu at
    block 64), including jumps far beyond 2^56; ragged last block.  At jump 40 every block-128
    item overshoots its reference and goes through the exact-max fallback passes."""
    heads, nb = 2, lay.NB
    q, k, v = qkv(1, lay.N, heads, d, seed=21, device="cuda")
    gain = torch.ones(lay.N, device="cuda")
    for c in range(nb):
        gain[c * 128:(c + 1) * 128] = 1.0 + jump * c / nb
    k = (k.float() * gain.view(1, -1, 1, 1)).to(torch.bfloat16)
    rng = np.random.default_rng(5)
    masks = (rng.random((heads, nb, nb)) < 0.6).astype(np.uint8)
    masks[:, :, 0] = 1  # every row starts from the low-score block
    masks[:, :, nb - 1] = 1  # and reaches the largest-score (ragged) block
    out, lse, _ = run_attention(csa, lay, q, k, v, masks=masks, lse=True)
    lse_np = lse.view(heads, lay.N).cpu().numpy()
    for h in range(heads):
        ref, ref_lse = oracle_head(lay, q, k, v, 0, h, mask=masks[h])
        assert_close(out[0, :, h].double().cpu().numpy(), ref, f"d{d} jump {jump} h{h}")
        assert np.abs(lse_np[h] - ref_lse).max() <= 1e-3 * max(1.0, np.abs(ref_lse).max())
    if lay.B == 128:  # the fixed-reference kernels
        n_fb = fallback_count(csa, q)
        assert (n_fb > 0) if jump > 10 else (n_fb == 0), n_fb


def test_attention_repetitive_block128(csa):
    """Anchor-row heads on the production kernel: k in {1, 2, 5, H}, ragged N, broadcast rows
    bitwise equal to their anchor row, a MASK head alongside."""
    lay = Layout(2, 9, 40, 128)
    q, k, v = qkv(1, lay.N, 2, 128, seed=44, device="cuda")
    rng = np.random.default_rng(2)
    masks = (rng.random((2, lay.NB, lay.NB)) < 0.5).astype(np.uint8)
    masks[:, np.arange(lay.NB), np.arange(lay.NB)] = 1
    for kA in (1, 2, 5, lay.H):
        out, lse, _ = run_attention(csa, lay, q, k, v, masks=masks, rep=[1], anchor_k=kA, lse=True)
        ref, ref_lse = oracle_head(lay, q, k, v, 0, 1, rep_k=kA)
        assert_close(out[0, :, 1].double().cpu().numpy(), ref, f"k={kA}")
        assert np.abs(lse.view(2, lay.N)[1].cpu().numpy() - ref_lse).max() <= 1e-3
        anchors = oracle.anchor_rows(lay.H, kA)
        o3 = out[0, :, 1].view(lay.F, lay.H, lay.W, -1)
        for i in range(lay.H):
            assert torch.equal(o3[:, i], o3[:, anchors[oracle.nearest_anchor(lay.H, kA, i)]])
        ref0, _ = oracle_head(lay, q, k, v, 0, 0, mask=masks[0])
        assert_close(out[0, :, 0].double().cpu().numpy(), ref0, "mask head")


def test_attention_tiny_repetitive(csa):
    cfg = CONFIGS["tiny"]
    lay = cfg.layout
    q, k, v = qkv(1, lay.N, 2, cfg.d, seed=4, device="cuda")
    for kA in (1, 2, 5, lay.H):
        out, _, _ = run_attention(csa, lay, q, k, v, rep=[1], anchor_k=kA)
        ref, _ = oracle_head(lay, q, k, v, 0, 1, rep_k=kA)
        o = out[0, :, 1].double().cpu().numpy()
        assert_close(o, ref, f"k={kA}")
        # broadcast rows are bitwise copies of their anchor row
        anchors = oracle.anchor_rows(lay.H, kA)
        o3 = out[0, :, 1].view(lay.F, lay.H, lay.W, -1)
        for i in range(lay.H):
            a = anchors[oracle.nearest_anchor(lay.H, kA, i)]
            assert torch.equal(o3[:, i], o3[:, a])
        ref0, _ = oracle_head(lay, q, k, v, 0, 0, mask=np.ones((lay.NB, lay.NB), np.uint8))
        assert_close(out[0, :, 0].double().cpu().numpy(), ref0, "dense head")


@pytest.mark.parametrize("lay,d", [(Layout(2, 5, 25, 64), 64), (Layout(2, 9, 40, 128), 128)])
def test_attention_batch2_shares_plan_and_is_deterministic(csa, lay, d):
    """Both kernels: attn.cu (B 64, dynamic and static assignment) and the production kernel
    (attn5.cu, B 128, d 128)."""
    q, k, v = qkv(2, lay.N, 3, d, seed=7, device="cuda")
    rng = np.random.default_rng(1)
    masks = (rng.random((3, lay.NB, lay.NB)) < 0.5).astype(np.uint8)
    masks[:, np.arange(lay.NB), np.arange(lay.NB)] = 1
    out, _, plan = run_attention(csa, lay, q, k, v, masks=masks, rep=[2], anchor_k=2)
    for order in (0, 1):
        out2, _, _ = run_attention(csa, lay, q, k, v, masks=masks, rep=[2], anchor_k=2, order=order)
        assert torch.equal(out, out2)  # item order never changes per-item arithmetic
    if lay.B == 64:  # static round-robin assignment (no workspace): same kernel, same bits
        static = csa.sparse_attn_fwd(q, k, v, plan, csa.build_work_list(plan, 0, 3), dynamic=False)
        assert torch.equal(out, static)
    again, _, _ = run_attention(csa, lay, q, k, v, masks=masks, rep=[2], anchor_k=2)
    assert torch.equal(out, again)  # run-to-run determinism (scheduler counters self-reset)
    for b in range(2):
        for h in range(3):
            ref, _ = oracle_head(lay, q, k, v, b, h, mask=masks[h], rep_k=2 if h == 2 else None)
            assert_close(out[b, :, h].double().cpu().numpy(), ref, f"b{b} h{h}")
        single, _, _ = run_attention(csa, lay, q[b:b + 1].contiguous(), k[b:b + 1].contiguous(),
                                     v[b:b + 1].contiguous(), masks=masks, rep=[2], anchor_k=2)
        assert torch.equal(single[0], out[b])


def _plan_from_masks(csa, lay, masks, rep, anchor_k, csr):
    heads = masks.shape[0]
    sim = torch.tensor([1.0 if h in rep else 0.0 for h in range(heads)], dtype=torch.float64,
                       device="cuda")
    return csa.compile_plan(lay, u16_dev(masks.astype(np.uint16)), 1, similarity=sim, gamma=0.87,
                            anchor_k=anchor_k, csr=csr)


@pytest.mark.parametrize("lay,d", [(Layout(2, 9, 40, 128), 128), (Layout(2, 9, 40, 128), 64),
                                   (Layout(2, 9, 40, 128, 80), 128), (Layout(2, 9, 40, 128, 192), 128),
                                   (Layout(2, 5, 25, 64), 64), (Layout(3, 7, 100, 128), 128)])
def test_intervals_only_plan_bitwise(csa, lay, d):
    """Intervals-only plans (no blk_idx; the kernels walk the 1-D skip list) give the
    CSR plan's outputs bit for bit on every attention kernel (attn5 d 128 / 64, attn_rect, attn at
    block 64), with a REPETITIVE head, batch 2, and through the exact-max fallback passes
    (scores growing 40x block by block); the validator accepts them; outputs match the oracle."""
    heads = 3
    q, k, v = qkv(2, lay.N, heads, d, seed=17, device="cuda")
    rng = np.random.default_rng(6)
    masks = (rng.random((heads, lay.NB, lay.NBK)) < 0.45).astype(np.uint8)
    masks[:, :, 0] = 1
    outs = {}
    for csr in (True, False):
        plan = _plan_from_masks(csa, lay, masks, [1], 2, csr)
        csa.validate_plan(plan)
        assert (plan.blk_idx.numel() > 0) == csr
        lse = torch.empty(2 * heads * lay.N, dtype=torch.float32, device="cuda")
        outs[csr] = (csa.sparse_attn_fwd(q, k, v, plan, csa.build_work_list(plan, 0, heads),
                                         lse_out=lse), lse)
    torch.cuda.synchronize()
    assert torch.equal(outs[True][0], outs[False][0])
    assert torch.equal(outs[True][1], outs[False][1])
    for h in (0, 2):
        ref, _ = oracle_head(lay, q, k, v, 1, h, mask=masks[h])
        assert_close(outs[False][0][1, :, h].double().cpu().numpy(), ref, f"h{h}")
    if lay.B == 128:  # overshooting rows through the fallback list, intervals-only plan
        gain = torch.ones(lay.N, device="cuda")
        for c in range(lay.NBK):
            gain[c * lay.Bkv:(c + 1) * lay.Bkv] = 1.0 + 40.0 * c / lay.NBK
        kj = (k.float() * gain.view(1, -1, 1, 1)).to(torch.bfloat16)
        res = []
        for csr in (True, False):
            plan = _plan_from_masks(csa, lay, masks, [], 2, csr)
            res.append(csa.sparse_attn_fwd(q, kj, v, plan, csa.build_work_list(plan, 0, heads)))
            torch.cuda.synchronize()
            assert fallback_count(csa, q) > 0
        assert torch.equal(res[0], res[1])
        ref, _ = oracle_head(lay, q, kj, v, 0, 1, mask=masks[1])
        assert_close(res[1][0, :, 1].double().cpu().numpy(), ref, "fallback")


def test_intervals_only_plan_full_size_and_validation(csa):
    """Wan 720p (generator-S masks, 4 anchor heads): the intervals-only plan is a fraction of the
    CSR plan's bytes and gives the same attention bit for bit; a corrupted interval (end moved
    by one) or a row count that no longer matches its intervals fails csa_validate_plan."""
    cfg = CONFIGS["wan720"]
    lay = cfg.layout
    q, k, v = qkv(1, lay.N, cfg.heads, cfg.d, seed=11, device="cuda")
    masks = inputs.synthetic_masks(lay, cfg.heads, cfg.sparsity, seed=0)
    rep = [0, 13, 26, 39]
    p_csr = _plan_from_masks(csa, lay, masks, rep, 5, True)
    p_ivl = _plan_from_masks(csa, lay, masks, rep, 5, False)
    csa.validate_plan(p_ivl)
    assert p_ivl.nbytes() < 0.3 * p_csr.nbytes(), (p_ivl.nbytes(), p_csr.nbytes())
    o1 = csa.sparse_attn_fwd(q, k, v, p_csr, csa.build_work_list(p_csr, 0, cfg.heads))
    o2 = csa.sparse_attn_fwd(q, k, v, p_ivl, csa.build_work_list(p_ivl, 0, cfg.heads))
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    iv = p_ivl.ivl.view(torch.int16)
    first_end = 1
    old = int(iv[first_end].item())
    iv[first_end] = old + 1                      # cover no longer equals the row count
    with pytest.raises(csa.CsaError, match="CORRUPT_PLAN"):
        csa.validate_plan(p_ivl)
    iv[first_end] = old
    csa.validate_plan(p_ivl)


@pytest.mark.parametrize("lay,peers", [(Layout(2, 9, 40, 128), 1), (Layout(2, 9, 40, 128), 2),
                                       (Layout(2, 9, 40, 128), 8), (Layout(3, 7, 100, 128), 4),
                                       (Layout(2, 9, 40, 128, 80), 4)])
def test_output_scatter_into_rank_buffers(csa, lay, peers):
    """csa_sparse_attn_fwd_scatter with P "virtual ranks" on one GPU (the kernel only sees a
    pointer table, local or peer-mapped alike): every output row lands in the receive buffer of
    the rank owning its token, at this rank's head columns, bit for bit the rows of
    csa_sparse_attn_fwd; other heads untouched.  REPETITIVE broadcast rows crossing shard
    boundaries, batch 2, and the exact-max fallback passes (scores growing 40x block by block:
    mode 1 parks each row's max in its first output row -- inside a rank's buffer -- and mode 2
    reads it back)."""
    hp, d, b = 3, 128, 2
    rank = peers - 1                                  # this rank's heads: [rank hp, rank hp + hp)
    H = hp * peers
    n_loc = lay.N // peers
    q, k, v = qkv(b, lay.N, hp, d, seed=23, device="cuda")
    rng = np.random.default_rng(3)
    masks = (rng.random((hp, lay.NB, lay.NBK)) < 0.5).astype(np.uint8)
    masks[:, :, 0] = 1
    for jump in (0.0, 40.0):
        kk = k
        if jump:
            gain = torch.ones(lay.N, device="cuda")
            for c in range(lay.NBK):
                gain[c * lay.Bkv:(c + 1) * lay.Bkv] = 1.0 + jump * c / lay.NBK
            kk = (k.float() * gain.view(1, -1, 1, 1)).to(torch.bfloat16)
        plan = _plan_from_masks(csa, lay, masks, [] if jump else [1], 2, True)
        work = csa.build_work_list(plan, 0, hp)
        ref = csa.sparse_attn_fwd(q, kk, v, plan, work)
        torch.cuda.synchronize()
        nfb = fallback_count(csa, q)
        bufs = [torch.zeros((b, n_loc, H, d), dtype=torch.bfloat16, device="cuda")
                for _ in range(peers)]
        ptrs = torch.tensor([t.data_ptr() + rank * hp * d * 2 for t in bufs], dtype=torch.int64,
                            device="cuda")
        csa.sparse_attn_fwd_scatter(q, kk, v, plan, work, ptrs, bufs[0])
        torch.cuda.synchronize()
        assert fallback_count(csa, q) == nfb and ((nfb > 0) == (jump > 0))
        for p_, t in enumerate(bufs):
            assert torch.equal(t[:, :, rank * hp:(rank + 1) * hp],
                               ref[:, p_ * n_loc:(p_ + 1) * n_loc]), (jump, p_)
            others = torch.cat([t[:, :, :rank * hp], t[:, :, (rank + 1) * hp:]], dim=2)
            assert not others.any()


def test_fused_out_layer_step_single_rank_nccl(csa):
    """ulysses.make_layer_step_fused_out through a real NCCL group and symmetric memory (one
    rank: the only peer is itself): the same output as the stacked-exchange layer step, bit for
    bit, over repeated steps (the barriers order the buffer's reuse)."""
    import socket

    import torch.distributed as dist

    from paper_2603_05503_b200 import ulysses
    lay = Layout(3, 7, 100, 128)
    H, d = 4, 128
    q, k, v = qkv(2, lay.N, H, d, seed=29, device="cuda")
    rng = np.random.default_rng(9)
    masks = (rng.random((H, lay.NB, lay.NB)) < 0.5).astype(np.uint8)
    masks[:, :, 0] = 1
    plan = _plan_from_masks(csa, lay, masks, [2], 2, True)
    work = csa.build_work_list(plan, 0, H)
    ref = csa.sparse_attn_fwd(q, k, v, plan, work)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        def attn(qv, kv, vv, ptrs, recv):
            csa.sparse_attn_fwd_scatter(qv, kv, vv, plan, work, ptrs, recv)

        step = ulysses.make_layer_step_fused_out(q, k, v, 1, attn)
        for _ in range(3):
            out = step()
            torch.cuda.synchronize()
            assert torch.equal(out, ref)
            out.zero_()
    finally:
        dist.destroy_process_group()


def sample_units(lay, heads, n, seed):
    rng = np.random.default_rng(seed)
    units = {(0, lay.NB - 1), (heads - 1, 0)}
    while len(units) < n:
        units.add((int(rng.integers(heads)), int(rng.integers(lay.NB))))
    return sorted(units)


@pytest.mark.parametrize("name", ["wan480", "wan720", "mochi"])
def test_attention_full_size_sampled(csa, name):
    """BASELINE configs at full size, bench launch configuration; oracle on sampled (h, r)
    (Mochi: generator-S masks at the paper's 69 % sparsity)."""
    cfg = CONFIGS[name]
    lay = cfg.layout
    q, k, v = qkv(1, lay.N, cfg.heads, cfg.d, seed=11, device="cuda")
    masks = inputs.synthetic_masks(lay, cfg.heads, cfg.sparsity or 0.69, seed=0)
    rep = [h for h in (3, 17, 29, 38) if h < cfg.heads]
    out, lse, plan = run_attention(csa, lay, q, k, v, masks=masks, rep=rep, anchor_k=5, lse=True)
    lse = lse.view(cfg.heads, lay.N).cpu().numpy()
    errs = []
    for h, r in sample_units(lay, cfg.heads, 10, seed=2):
        rows = (r * lay.B, min((r + 1) * lay.B, lay.N))
        ref, ref_lse = oracle_head(lay, q, k, v, 0, h, mask=masks[h],
                                   rep_k=5 if h in rep else None, rows=rows)
        got = out[0, rows[0]:rows[1], h].double().cpu().numpy()
        assert_close(got, ref, f"h{h} r{r}")
        assert np.abs(lse[h, rows[0]:rows[1]] - ref_lse).max() <= 1e-3
        errs.append(np.abs(got - ref).max())
    assert torch.isfinite(out).all()
    if cfg.d == 128:
        assert fallback_count(csa, q) == 0  # realistic rows never overshoot the reference max


def test_attention_wan720_structured_peaked_sampled(csa):
    """Wan 720p at full size on generator-G Q/K (peak-logit scale alpha up to 1.6, sink keys,
    two repetitive heads), plan CALIBRATED from the same prompt (a2-a6 through the C ABI, eps of
    t = 25 of 50), production launch.  Rows keep block 0 (the sinks), so their first kept tile
    -- the fixed softmax reference of reading Q29 -- sits far below the row's peak near the
    diagonal: this exercises the shift at full size with peaked logits, not just i.i.d. scores.
    Oracle on sampled units incl. the ragged last block and anchor rows."""
    cfg = CONFIGS["wan720"]
    lay = cfg.layout
    heads = 8
    alphas = np.linspace(0.8, 1.6, heads)
    q, k, v = inputs.structured_qk(lay, heads, 128, 9, 0, alpha=alphas, repetitive=(2, 5),
                                   device="cuda")
    nb = lay.NB
    counts = u16_zeros(heads * nb * nb)
    lse_c = torch.empty(heads * lay.N, dtype=torch.float32, device="cuda")
    eps = oracle.epsilon(25, 50, oracle.A_of_N(lay.N), 0.99, 16)
    csa.calib_accumulate(lay, q, k, eps, counts, lse_out=lse_c)
    sim = torch.zeros(heads, dtype=torch.float64, device="cuda")
    csa.spatial_similarity(lay, q, k, lse_c, 5, sim)
    s = sim / float(lay.F * lay.H)
    plan = csa.compile_plan(lay, counts, 1, similarity=s, gamma=0.87, anchor_k=5)
    work = csa.build_work_list(plan, 0, heads)
    lse = torch.empty(heads * lay.N, dtype=torch.float32, device="cuda")
    out = csa.sparse_attn_fwd(q, k, v, plan, work, lse_out=lse)
    torch.cuda.synchronize()
    kinds = plan.kind_host
    assert kinds[2] == 1 and kinds[5] == 1, kinds   # the generated repetitive heads are detected
    cnt = u16_np(counts).reshape(heads, nb, nb)
    masks = (cnt >= 1).astype(np.uint8)
    for h in range(heads):   # the compiler's row repair (reading Q7) never triggers here
        if not kinds[h]:
            assert masks[h].sum(axis=1).min() >= 1
    lse = lse.view(heads, lay.N).cpu().numpy()
    units = [(0, 0), (0, nb - 1), (2, 0), (5, nb - 1), (7, nb // 2), (7, nb - 1)]
    rng = np.random.default_rng(4)
    units += [(int(rng.integers(heads)), int(rng.integers(nb))) for _ in range(8)]
    for h, r in units:
        rows = (r * lay.B, min((r + 1) * lay.B, lay.N))
        rep_k = 5 if kinds[h] else None
        ref, ref_lse = oracle_head(lay, q, k, v, 0, h, mask=masks[h], rep_k=rep_k, rows=rows)
        got = out[0, rows[0]:rows[1], h].double().cpu().numpy()
        assert_close(got, ref, f"h{h} r{r}")
        assert np.abs(lse[h, rows[0]:rows[1]] - ref_lse).max() <= 1e-3, (h, r)
    assert torch.isfinite(out).all()


# ---------------------------------------------------------------- a2-a5 calibration
@pytest.mark.parametrize("lay,heads,d", [(Layout(2, 5, 25, 64), 2, 64), (Layout(4, 8, 8, 64), 1, 64),
                                         (Layout(2, 9, 40, 128), 2, 128),
                                         (Layout(2, 9, 40, 128, 80), 2, 128),
                                         (Layout(2, 9, 40, 128, 192), 2, 128),
                                         (Layout(3, 7, 100, 128, 64), 2, 128)])
@pytest.mark.parametrize("single_pass", [True, False])
def test_calibration_against_oracle(csa, lay, heads, d, single_pass):
    q, k, _ = inputs.structured_qk(lay, heads, d, head_seed=1, prompt_seed=2, alpha=1.0,
                                   device="cuda")
    nb, nbk = lay.NB, lay.NBK
    eps = 0.9
    counts = u16_zeros(heads * nb * nbk)
    counts_np = np.zeros((heads, nb, nbk), np.uint16)
    energy = torch.empty(heads * nb * nbk, dtype=torch.float32, device="cuda")
    lse_out = torch.empty(heads * lay.N, dtype=torch.float32, device="cuda")
    scale = 1.0 / np.sqrt(d)
    for prompt in range(3):  # accumulate over prompts: integer counts exact
        q, k, _ = inputs.structured_qk(lay, heads, d, 1, prompt, alpha=1.0, device="cuda")
        csa.calib_accumulate(lay, q, k, eps, counts, energy_out=energy, lse_out=lse_out,
                             single_pass=single_pass)
        torch.cuda.synchronize()
        E = energy.view(heads, nb, nbk).double().cpu().numpy()
        lg = lse_out.view(heads, lay.N).double().cpu().numpy()
        for h in range(heads):
            qh, kh = head64(q, 0, h), head64(k, 0, h)
            ref_lse = oracle.row_lse(qh, kh, scale)
            assert np.abs(lg[h] - ref_lse).max() <= 1e-3
            E_ref = oracle.block_energy(qh, kh, scale, lay.B, block_kv=lay.BK or None)
            assert np.abs(E[h] - E_ref).max() <= 5e-5
            assert np.abs(E[h].sum(1) - 1).max() <= 1e-4
            for r in range(nb):
                oracle.accumulate(oracle.select(E[h, r], eps), counts_np[h, r])
                # SURVEY 8.4 contract 4: the oracle's selection on its OWN fp64 E may differ
                # from the GPU's only on borderline rows (cut within 1e-5 of eps, or a tie
                # within 1e-5 at the cut)
                if not np.array_equal(oracle.select(E_ref[r], eps), oracle.select(E[h, r], eps)):
                    assert _borderline(E_ref[r], eps), (h, r)
        assert np.array_equal(u16_np(counts).reshape(heads, nb, nbk), counts_np)
    # LSE supplied from outside (the dense run's statistic) gives the same decisions on this E
    counts2 = u16_zeros(heads * nb * nbk)
    csa.calib_accumulate(lay, q, k, eps, counts2, lse_in=lse_out, energy_out=energy)
    torch.cuda.synchronize()
    E2 = energy.view(heads, nb, nbk).double().cpu().numpy()
    c2 = u16_np(counts2).reshape(heads, nb, nbk)
    for h in range(heads):
        for r in range(nb):
            assert np.array_equal(oracle.select(E2[h, r], eps), c2[h, r])


def _borderline(e_row, eps, tol=1e-5):
    e = np.sort(np.asarray(e_row, np.float64))[::-1]
    cs = np.cumsum(e)
    k = int(np.searchsorted(cs, eps))  # first prefix reaching eps
    near_cut = np.min(np.abs(cs - eps)) < tol
    tie = k + 1 < len(e) and abs(e[min(k, len(e) - 1)] - e[k + 1]) < tol
    return bool(near_cut or tie)


@pytest.mark.parametrize("name", ["wan480", "wan720"])
def test_calibration_full_size_sampled(csa, name):
    cfg = CONFIGS[name]
    lay = cfg.layout
    heads = 4
    q, k, _ = inputs.structured_qk(lay, heads, cfg.d, 5, 0, alpha=[0.8, 1.0, 1.2, 1.5],
                                   repetitive=(2,), device="cuda")
    nb = lay.NB
    counts = u16_zeros(heads * nb * nb)
    energy = torch.empty(heads * nb * nb, dtype=torch.float32, device="cuda")
    eps = oracle.epsilon(25, 50, oracle.A_of_N(lay.N), 0.99, 16)
    csa.calib_accumulate(lay, q, k, eps, counts, energy_out=energy)
    torch.cuda.synchronize()
    E = energy.view(heads, nb, nb).double().cpu().numpy()
    cnt = u16_np(counts).reshape(heads, nb, nb)
    scale = 1.0 / np.sqrt(cfg.d)
    for h in range(heads):
        for r in range(nb):  # bit-exact selection on the GPU's own E, every row
            assert np.array_equal(oracle.select(E[h, r], eps), cnt[h, r])
    for h, r in ((0, 0), (3, nb - 1), (1, nb // 2)):
        qh, kh = head64(q, 0, h), head64(k, 0, h)
        E_ref = oracle.block_energy(qh, kh, scale, lay.B, block_rows=(r, r + 1))
        assert np.abs(E[h, r] - E_ref[0]).max() <= 5e-5
        if not np.array_equal(oracle.select(E_ref[0], eps), cnt[h, r]):  # contract 4
            assert _borderline(E_ref[0], eps), (h, r)


# ---------------------------------------------------------------- f1 spatial similarity
def _gpu_similarity(csa, lay, q, k, kA, reps=1):
    heads = q.shape[2]
    nb = lay.NB
    lse = torch.empty(heads * lay.N, dtype=torch.float32, device="cuda")
    counts = u16_zeros(heads * nb * nb)
    csa.calib_accumulate(lay, q, k, 0.9, counts, lse_out=lse)   # the pass's own LSE
    sim = torch.zeros(heads, dtype=torch.float64, device="cuda")
    cos = torch.empty(heads * lay.F * lay.H, dtype=torch.float32, device="cuda")
    for _ in range(reps):
        csa.spatial_similarity(lay, q, k, lse, kA, sim, cos_out=cos)
    torch.cuda.synchronize()
    return sim.cpu().numpy(), cos.view(heads, lay.F, lay.H).double().cpu().numpy()


@pytest.mark.parametrize("lay,heads,d", [(Layout(2, 5, 25, 64), 2, 64), (Layout(2, 9, 40, 128), 2, 128)])
@pytest.mark.parametrize("kind", ["random", "structured"])
def test_spatial_similarity_against_oracle(csa, lay, heads, d, kind):
    if kind == "random":
        q, k, _ = qkv(1, lay.N, heads, d, seed=41, device="cuda")
    else:
        q, k, _ = inputs.structured_qk(lay, heads, d, 3, 1, alpha=[0.9, 1.4], repetitive=(1,),
                                       device="cuda")
    scale = 1.0 / np.sqrt(d)
    for kA in (1, 2, lay.H):
        sim, cos = _gpu_similarity(csa, lay, q, k, kA)
        for h in range(heads):
            qh, kh = head64(q, 0, h), head64(k, 0, h)
            ref = np.array([[oracle.spatial_cos(lay.F, lay.H, lay.W, qh, kh, scale, kA, f, i)
                             for i in range(lay.H)] for f in range(lay.F)])
            assert np.abs(cos[h] - ref).max() <= 2e-5, (kind, kA, h)
            assert abs(sim[h] - cos[h].sum()) <= 1e-7 * lay.F * lay.H  # cos_out is fp32
            assert abs(sim[h] / (lay.F * lay.H) - ref.mean()) <= 2e-5
        if kA == lay.H:
            assert np.abs(cos - 1.0).max() <= 1e-5  # every row is its own anchor


@pytest.mark.parametrize("lay,d", [(Layout(2, 9, 40, 128), 128), (Layout(2, 9, 40, 128), 64),
                                   (Layout(3, 7, 100, 128), 128), (Layout(1, 3, 40, 128), 128),
                                   (Layout(1, 2, 30, 128), 128),
                                   (Layout(2, 5, 25, 64), 64), (Layout(2, 9, 40, 128, 80), 128)])
def test_calib_sim_fused_against_oracle(csa, lay, d):
    """csa_calib_accumulate_sim (a2-a5 + f1 in one pass; calibsim.cu at block 128 x 128, the two
    calls' kernels in sequence otherwise): E, LSE, the selection and cos(f, i) against the fp64
    oracle, and the same outputs as calib_accumulate + spatial_similarity within fp32 rounding
    order.  N_B = 1 (one ragged block: group 1 has no key tile; N = 60: chunks past the last
    key fully masked), odd N_B, ragged N, d 64, block 64 and B_kv = 80."""
    heads, kA = 2, 2
    q, k, _ = inputs.structured_qk(lay, heads, d, 3, 1, alpha=[0.9, 1.4], repetitive=(1,),
                                   device="cuda")
    nb, nbk = lay.NB, lay.NBK
    eps = oracle.epsilon(20, 50, oracle.A_of_N(lay.N), 0.99, 16)
    cnt_f = u16_zeros(heads * nb * nbk)
    E_f = torch.empty(heads * nb * nbk, dtype=torch.float32, device="cuda")
    lse_f = torch.empty(heads * lay.N, dtype=torch.float32, device="cuda")
    sim_f = torch.zeros(heads, dtype=torch.float64, device="cuda")
    cos_f = torch.empty(heads * lay.F * lay.H, dtype=torch.float32, device="cuda")
    csa.calib_accumulate_sim(lay, q, k, eps, cnt_f, kA, sim_f, energy_out=E_f, lse_out=lse_f,
                             cos_out=cos_f)
    # the two-call sequence on the same prompt
    cnt_s = u16_zeros(heads * nb * nbk)
    E_s = torch.empty_like(E_f)
    lse_s = torch.empty_like(lse_f)
    sim_s = torch.zeros_like(sim_f)
    cos_s = torch.empty_like(cos_f)
    csa.calib_accumulate(lay, q, k, eps, cnt_s, energy_out=E_s, lse_out=lse_s)
    csa.spatial_similarity(lay, q, k, lse_s, kA, sim_s, cos_out=cos_s)
    torch.cuda.synchronize()
    E = E_f.view(heads, nb, nbk).double().cpu().numpy()
    cnt = u16_np(cnt_f).reshape(heads, nb, nbk)
    cos = cos_f.view(heads, lay.F, lay.H).double().cpu().numpy()
    assert np.abs(E - E_s.view(heads, nb, nbk).double().cpu().numpy()).max() <= 5e-6
    assert np.abs(lse_f.cpu().numpy() - lse_s.cpu().numpy()).max() <= 1e-4
    assert np.abs(cos - cos_s.view(heads, lay.F, lay.H).double().cpu().numpy()).max() <= 2e-6
    scale = 1.0 / np.sqrt(d)
    lse = lse_f.view(heads, lay.N).cpu().numpy()
    for h in range(heads):
        qh, kh = head64(q, 0, h), head64(k, 0, h)
        E_ref = oracle.block_energy(qh, kh, scale, lay.B, block_kv=lay.BK or None)
        assert np.abs(E[h] - E_ref).max() <= 5e-5, h
        for r in range(nb):  # bit-exact selection on the pass's own E
            assert np.array_equal(oracle.select(E[h, r], eps), cnt[h, r]), (h, r)
        assert np.abs(lse[h] - oracle.row_lse(qh, kh, scale)).max() <= 1e-3
        ref = np.array([[oracle.spatial_cos(lay.F, lay.H, lay.W, qh, kh, scale, kA, f, i)
                         for i in range(lay.H)] for f in range(lay.F)])
        assert np.abs(cos[h] - ref).max() <= 2e-5, h
        assert abs(sim_f[h].item() / (lay.F * lay.H) - ref.mean()) <= 2e-5


@pytest.mark.parametrize("name", ["wan720", "mochi"])
def test_calib_sim_fused_full_size_sampled(csa, name):
    """Full-size fused pass (generator-G Q/K, one repetitive head): every row's selection
    bit-exact on the pass's own E, sampled E rows and cos(f, i) against the oracle, and all cos
    within fp32 rounding of the two-call sequence."""
    cfg = CONFIGS[name]
    lay = cfg.layout
    heads, kA = 4, 5
    q, k, _ = inputs.structured_qk(lay, heads, cfg.d, 5, 0, alpha=[0.8, 1.0, 1.2, 1.5],
                                   repetitive=(2,), device="cuda")
    nb = lay.NB
    eps = oracle.epsilon(25, 50, oracle.A_of_N(lay.N), 0.99, 16)
    counts = u16_zeros(heads * nb * nb)
    energy = torch.empty(heads * nb * nb, dtype=torch.float32, device="cuda")
    sim = torch.zeros(heads, dtype=torch.float64, device="cuda")
    cos_f = torch.empty(heads * lay.F * lay.H, dtype=torch.float32, device="cuda")
    csa.calib_accumulate_sim(lay, q, k, eps, counts, kA, sim, energy_out=energy, cos_out=cos_f)
    lse_s = torch.empty(heads * lay.N, dtype=torch.float32, device="cuda")
    csa.calib_accumulate(lay, q, k, eps, u16_zeros(heads * nb * nb), lse_out=lse_s)
    cos_s = torch.empty_like(cos_f)
    csa.spatial_similarity(lay, q, k, lse_s, kA, torch.zeros_like(sim), cos_out=cos_s)
    torch.cuda.synchronize()
    E = energy.view(heads, nb, nb).double().cpu().numpy()
    cnt = u16_np(counts).reshape(heads, nb, nb)
    cos = cos_f.view(heads, lay.F, lay.H).double().cpu().numpy()
    assert np.abs(cos - cos_s.view(heads, lay.F, lay.H).double().cpu().numpy()).max() <= 2e-6
    for h in range(heads):
        for r in range(nb):
            assert np.array_equal(oracle.select(E[h, r], eps), cnt[h, r])
    scale = 1.0 / np.sqrt(cfg.d)
    for h, r in ((0, 0), (3, nb - 1), (2, nb // 2)):
        qh, kh = head64(q, 0, h), head64(k, 0, h)
        E_ref = oracle.block_energy(qh, kh, scale, lay.B, block_rows=(r, r + 1))
        assert np.abs(E[h, r] - E_ref[0]).max() <= 5e-5
    for h, f, i in ((0, 0, 0), (2, lay.F - 1, lay.H // 2), (3, lay.F // 2, lay.H - 1)):
        qh, kh = head64(q, 0, h), head64(k, 0, h)
        ref = oracle.spatial_cos(lay.F, lay.H, lay.W, qh, kh, scale, kA, f, i)
        assert abs(cos[h, f, i] - ref) <= 2e-5, (h, f, i)


def test_spatial_similarity_repetitive_structure_and_accumulation(csa):
    lay = Layout(2, 9, 40, 128)
    heads = 2
    q, k, _ = qkv(1, lay.N, heads, 128, seed=43, device="cuda")
    # queries independent of the spatial row: P^(f,i) = P^(f,a(i)) -> cos = 1 (Obs. 4)
    q3 = q.view(1, lay.F, lay.H, lay.W, heads, 128)
    qr = q3[:, :, :1].expand(-1, -1, lay.H, -1, -1, -1).reshape(1, lay.N, heads, 128).contiguous()
    sim, cos = _gpu_similarity(csa, lay, qr, k, 3)
    assert np.abs(cos - 1.0).max() <= 1e-5
    # sim_sum accumulates across prompts; repeated runs are bitwise identical
    s1, c1 = _gpu_similarity(csa, lay, q, k, 3, reps=1)
    s2, c2 = _gpu_similarity(csa, lay, q, k, 3, reps=2)
    assert np.array_equal(c1, c2)
    assert np.array_equal(2 * s1, s2)


def test_spatial_similarity_wan480_sampled(csa):
    cfg = CONFIGS["wan480"]
    lay = cfg.layout
    heads = 2
    q, k, _ = inputs.structured_qk(lay, heads, cfg.d, 5, 0, alpha=[1.0, 1.3], repetitive=(1,),
                                   device="cuda")
    sim, cos = _gpu_similarity(csa, lay, q, k, 5)
    scale = 1.0 / np.sqrt(cfg.d)
    for h, f, i in ((0, 0, 0), (0, 20, 29), (1, 7, 13), (1, 0, 3)):
        qh, kh = head64(q, 0, h), head64(k, 0, h)
        ref = oracle.spatial_cos(lay.F, lay.H, lay.W, qh, kh, scale, 5, f, i)
        assert abs(cos[h, f, i] - ref) <= 2e-5, (h, f, i)
    assert sim[1] / (lay.F * lay.H) > sim[0] / (lay.F * lay.H)  # the repetitive head scores higher


# ---------------------------------------------------------------- f2 plan compaction
def _row_intervals(mask_row):
    ivl, c, nb = [], 0, len(mask_row)
    while c < nb:
        if mask_row[c]:
            s = c
            while c < nb and mask_row[c]:
                c += 1
            ivl.append((s, c))
        else:
            c += 1
    return ivl


@pytest.mark.parametrize("lay", [Layout(2, 5, 25, 64), Layout(21, 30, 52, 128),
                                 Layout(21, 30, 52, 128, 80)])
@pytest.mark.parametrize("pct", [100.0, 90.0, 50.0])
def test_merge_intervals_bit_exact(csa, lay, pct):
    nbq, nb, cells = lay.NB, lay.NBK, 4
    counts_np = inputs.random_counts(nbq, cells, 8, seed=nb + int(pct), nbk=nb)
    counts_np[2][:, ::2] = 8  # alternating rows: the widest rows
    sim = torch.tensor([0.0, 0.0, 0.0, 1.0], dtype=torch.float64, device="cuda")  # cell 3 REPETITIVE
    counts = u16_dev(counts_np)
    plan = csa.compile_plan(lay, counts, 4, similarity=sim, anchor_k=min(5, lay.H))
    bits = unpack_bits(plan.mask_bits.cpu().numpy(), nb).reshape(cells, nbq, nb)
    widths = [len(_row_intervals(bits[c, r])) for c in range(3) for r in range(nbq)]
    target_ref = oracle.percentile_nearest_rank(widths, pct)
    target, added = csa.merge_intervals(plan, counts, 4, pct)
    torch.cuda.synchronize()
    assert int(target.item()) == target_ref
    got = u16_np(counts).reshape(cells, nbq, nb)
    ref = counts_np.copy()
    added_ref = 0
    for c in range(3):
        for r in range(nbq):
            merged, add = oracle.merge_row(_row_intervals(bits[c, r]), max(target_ref, 1))
            added_ref += add
            kept = np.zeros(nb, bool)
            for s0, e0 in merged:
                kept[s0:e0] = True
            filled = kept & ~bits[c, r].astype(bool)
            ref[c, r][filled] = 4
    assert np.array_equal(got, ref)
    assert int(added.item()) == added_ref
    # recompiled plan: every row within the target, kept sets supersets
    plan2 = csa.compile_plan(lay, counts, 4, similarity=sim, anchor_k=min(5, lay.H))
    bits2 = unpack_bits(plan2.mask_bits.cpu().numpy(), nb).reshape(cells, nbq, nb)
    assert (bits2[:3] >= bits[:3]).all()
    irp = plan2.ivl_row_ptr.cpu().numpy().reshape(cells, nbq + 1)
    assert np.diff(irp[:3], axis=1).max() <= max(target_ref, 1)


def test_share_timesteps_bit_exact(csa):
    lay = Layout(21, 30, 52, 128)
    nb, T, G = lay.NB, 6, 3
    rng = np.random.default_rng(12)
    base = inputs.random_counts(nb, G, 8, seed=77)
    counts_np = np.zeros((T, G, nb, nb), np.uint16)
    for t in range(T):  # later timesteps drift less: the late ones become near-identical
        noise = rng.random((G, nb, nb)) < 0.2 * (T - t) / T
        counts_np[t] = np.where(noise, 8 - base, base)
    sim = torch.zeros(T * G, dtype=torch.float64, device="cuda")
    sim[(T - 1) * G + 2] = 1.0  # one REPETITIVE cell (t = T-1, g = 2)
    counts = u16_dev(counts_np.reshape(-1, nb, nb))
    plan = csa.compile_plan(lay, counts, 4, similarity=sim, anchor_k=5)
    bits = unpack_bits(plan.mask_bits.cpu().numpy(), nb).reshape(T, G, nb, nb)
    kind = plan.kind.cpu().numpy().reshape(T, G)
    tau = 0.6
    cluster, iou = csa.share_timesteps(plan, counts, G, T, 4, tau)
    torch.cuda.synchronize()
    iou = iou.cpu().numpy()
    cluster = cluster.cpu().numpy()
    got = u16_np(counts).reshape(T, G, nb, nb)
    for g in range(G):
        ref_iou = np.empty((T, T))
        for t1 in range(T):
            for t2 in range(T):
                rep = kind[t1, g] or kind[t2, g]
                ref_iou[t1, t2] = -1.0 if rep else oracle.skipped_iou(bits[t1, g], bits[t2, g])
        assert np.array_equal(iou[g], ref_iou)  # exact ratio of integers
        ref_cl = oracle.cluster_timesteps(ref_iou, tau)
        assert np.array_equal(cluster[g], ref_cl)
        for t in range(T):
            if kind[t, g]:
                assert np.array_equal(got[t, g], counts_np[t, g])  # untouched
                continue
            members = [u for u in range(T) if ref_cl[u] == ref_cl[t] and not kind[u, g]]
            shared = np.zeros((nb, nb), bool)
            for u in members:
                shared |= bits[u, g].astype(bool)
            assert np.array_equal(got[t, g], np.where(shared, 4, 0).astype(np.uint16))
    assert len(set(cluster[0].tolist())) < T  # the late, near-identical timesteps share


# ---------------------------------------------------------------- e: head sharding invariant
@pytest.mark.parametrize("world", [2, 4])
def test_head_sharded_launches_are_bitwise_equal_to_the_full_launch(csa, world):
    """per-head outputs are bit-identical for any head partition P -- each rank's
    launch sees only its heads' cells and a head-sliced (received) copy of Q, K, V."""
    lay = Layout(21, 30, 52, 128)
    heads = 8
    q, k, v = qkv(1, lay.N, heads, 128, seed=61, device="cuda")
    rng = np.random.default_rng(4)
    masks = (rng.random((heads, lay.NB, lay.NB)) < 0.3).astype(np.uint8)
    masks[:, np.arange(lay.NB), np.arange(lay.NB)] = 1
    rep = [3]
    full, _, _ = run_attention(csa, lay, q, k, v, masks=masks, rep=rep, anchor_k=5)
    hp = heads // world
    for r in range(world):
        sl = slice(r * hp, (r + 1) * hp)
        part, _, _ = run_attention(csa, lay, q[:, :, sl].contiguous(), k[:, :, sl].contiguous(),
                                   v[:, :, sl].contiguous(), masks=masks[sl],
                                   rep=[h - r * hp for h in rep if r * hp <= h < (r + 1) * hp],
                                   anchor_k=5)
        assert torch.equal(part, full[:, :, sl])


@pytest.mark.parametrize("batch", [1, 2])
def test_exchange_layout_views_read_and_written_in_place(csa, batch):
    """The stacked Ulysses exchange (ulysses.LayerExchange) hands the kernel Q, K, V as strided
    views of one receive buffer [N, B, 3, H/P, d] (batch inside the token) and lets it write O
    into the send buffer of the return exchange [N, B, H/P, d]: the TMA maps and the epilogue
    take those strides, and the result is the contiguous call's bit for bit."""
    from paper_2603_05503_b200 import ulysses

    lay = Layout(21, 30, 52, 128)
    heads = 4
    q, k, v = qkv(batch, lay.N, heads, 128, seed=62, device="cuda")
    rng = np.random.default_rng(5)
    masks = (rng.random((heads, lay.NB, lay.NB)) < 0.3).astype(np.uint8)
    masks[:, np.arange(lay.NB), np.arange(lay.NB)] = 1
    ref, _, plan = run_attention(csa, lay, q, k, v, masks=masks, rep=[1], anchor_k=5)
    ex = ulysses.LayerExchange(batch, lay.N, 1, heads, 128, torch.bfloat16, "cuda")
    ex.pack((q, k, v), 1, heads, 0)
    ex.recv.copy_(ex.send)                       # a world-1 exchange
    qs, ks, vs, os_ = ex.qkv(0), ex.qkv(1), ex.qkv(2), ex.out_view()
    assert qs.stride() == (3 * heads * 128, 3 * batch * heads * 128, 128, 1)
    csa.sparse_attn_fwd(qs, ks, vs, plan, csa.build_work_list(plan, 0, heads), out=os_)
    torch.cuda.synchronize()
    assert torch.equal(os_, ref)


def test_host_streaming_api_equals_device_call(csa):
    """csa.sparse_attn_fwd_host (pinned host in/out, head chunks with overlapped copies) gives
    the device call's output bit for bit (per-head arithmetic is schedule- and chunk-free)."""
    lay = Layout(21, 30, 52, 128)
    heads = 10
    q, k, v = qkv(1, lay.N, heads, 128, seed=62, device="cuda")
    rng = np.random.default_rng(6)
    masks = (rng.random((heads, lay.NB, lay.NB)) < 0.3).astype(np.uint8)
    masks[:, np.arange(lay.NB), np.arange(lay.NB)] = 1
    ref, _, plan = run_attention(csa, lay, q, k, v, masks=masks, rep=[4], anchor_k=5)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    for chunk in (3, 4, 10):
        ho = torch.zeros(q.shape, dtype=q.dtype).pin_memory()
        csa.sparse_attn_fwd_host(hq, hk, hv, plan, ho, heads_per_chunk=chunk)
        torch.cuda.synchronize()
        assert torch.equal(ho, ref.cpu()), chunk


# ---------------------------------------------------------------- f3: non-square B_q x B_kv
BKV_ALL = [64, 80, 96, 112, 144, 160, 176, 192]
# Table tab:block_size_ablation: mask sparsity per B_q x B_kv at Wan 480p
PAPER_SPARSITY = {64: 0.649, 80: 0.646, 96: 0.641, 128: 0.634, 144: 0.631, 176: 0.625, 192: 0.621}


@pytest.mark.parametrize("lay", [Layout(2, 9, 40, 128, 80), Layout(3, 7, 100, 128, 176),
                                 Layout(21, 30, 52, 128, 64)])
def test_rect_plan_compile_bit_exact(csa, lay):
    """a6 on a B_q x B_kv grid (rows N_B query blocks, columns N_Bkv key blocks)."""
    counts = inputs.random_counts(lay.NB, 5, 64, seed=lay.NBK, nbk=lay.NBK)
    counts[1] = 0
    counts[2] = 64
    counts[3] = 0
    counts[3][:, ::2] = 40
    check_plan_against_oracle(csa, lay, counts, 32)
    check_plan_against_oracle(csa, lay, counts, 32, sim=[0.5, 0.87, 0.9, 1.0, 0.0],
                              anchor_k=min(5, lay.H))


@pytest.mark.parametrize("bkv,d", [(b, 128) for b in BKV_ALL] + [(64, 64), (128, 64), (176, 64)])
def test_rect_attention_against_oracle(csa, bkv, d):
    """Every B_kv kernel instance (head_dim 128; head_dim 64 at 64, square 128 -- the d = 64 path
    -- and 176): ragged N (N_Bkv ragged for most B_kv), random MASK heads, an anchor head,
    batch 2 sharing the plan, lse; outputs vs the fp64 oracle on the same grid."""
    lay = Layout(2, 9, 40, 128, 0 if bkv == 128 else bkv)  # N = 720
    heads = 3
    q, k, v = qkv(2, lay.N, heads, d, seed=bkv + d, device="cuda")
    rng = np.random.default_rng(bkv)
    masks = (rng.random((heads, lay.NB, lay.NBK)) < 0.5).astype(np.uint8)
    masks[:, :, -1] = 1  # the ragged last key block
    out, lse, _ = run_attention(csa, lay, q, k, v, masks=masks, rep=[2], anchor_k=2, lse=True)
    lse = lse.view(2, heads, lay.N).cpu().numpy()
    for b in range(2):
        for h in range(heads):
            ref, ref_lse = oracle_head(lay, q, k, v, b, h, mask=masks[h],
                                       rep_k=2 if h == 2 else None)
            assert_close(out[b, :, h].double().cpu().numpy(), ref, f"B_kv {bkv} b{b} h{h}")
            assert np.abs(lse[b, h] - ref_lse).max() <= 1e-3
    again, _, _ = run_attention(csa, lay, q, k, v, masks=masks, rep=[2], anchor_k=2)
    assert torch.equal(out, again)
    assert fallback_count(csa, q) == 0


@pytest.mark.parametrize("bkv,d", [(80, 128), (192, 128), (128, 64)])
def test_rect_attention_overflow_fallback(csa, bkv, d):
    """Scores growing 40x block by block overshoot the first tile's reference max by far more
    than 2^56: those items go through the exact-row-max fallback (modes 1, 2) and still match."""
    lay = Layout(2, 9, 40, 128, 0 if bkv == 128 else bkv)
    heads = 2
    q, k, v = qkv(1, lay.N, heads, d, seed=21, device="cuda")
    gain = torch.ones(lay.N, device="cuda")
    for c in range(lay.NBK):
        gain[c * bkv:(c + 1) * bkv] = 1.0 + 40.0 * c / lay.NBK
    k = (k.float() * gain.view(1, -1, 1, 1)).to(torch.bfloat16)
    rng = np.random.default_rng(5)
    masks = (rng.random((heads, lay.NB, lay.NBK)) < 0.6).astype(np.uint8)
    masks[:, :, 0] = 1
    masks[:, :, -1] = 1
    out, lse, _ = run_attention(csa, lay, q, k, v, masks=masks, lse=True)
    assert fallback_count(csa, q) > 0
    lse_np = lse.view(heads, lay.N).cpu().numpy()
    for h in range(heads):
        ref, ref_lse = oracle_head(lay, q, k, v, 0, h, mask=masks[h])
        assert_close(out[0, :, h].double().cpu().numpy(), ref, f"B_kv {bkv} h{h}")
        assert np.abs(lse_np[h] - ref_lse).max() <= 1e-3 * max(1.0, np.abs(ref_lse).max())


@pytest.mark.parametrize("bkv", [64, 176])
def test_rect_attention_wan480_sampled(csa, bkv):
    """Wan 480p at full size on the B_q x B_kv grid at the paper's Table sparsity for that block
    size, 4 anchor heads, bench launch configuration; oracle on sampled units."""
    cfg = CONFIGS["wan480"]
    lay = Layout(cfg.layout.F, cfg.layout.H, cfg.layout.W, 128, bkv)
    q, k, v = qkv(1, lay.N, cfg.heads, cfg.d, seed=11, device="cuda")
    masks = inputs.synthetic_masks(lay, cfg.heads, PAPER_SPARSITY[bkv], seed=0)
    rep = [3, 17, 29, 38]
    out, lse, _ = run_attention(csa, lay, q, k, v, masks=masks, rep=rep, anchor_k=5, lse=True)
    lse = lse.view(cfg.heads, lay.N).cpu().numpy()
    for h, r in sample_units(lay, cfg.heads, 8, seed=4):
        rows = (r * lay.B, min((r + 1) * lay.B, lay.N))
        ref, ref_lse = oracle_head(lay, q, k, v, 0, h, mask=masks[h],
                                   rep_k=5 if h in rep else None, rows=rows)
        assert_close(out[0, rows[0]:rows[1], h].double().cpu().numpy(), ref, f"h{h} r{r}")
        assert np.abs(lse[h, rows[0]:rows[1]] - ref_lse).max() <= 1e-3
    assert torch.isfinite(out).all()
    assert fallback_count(csa, q) == 0


# ---------------------------------------------------------------- f4: dictionary + denoise step
def test_denoise_step_dictionary_graph_and_oracle(csa):
    """Distilled 4-step schedule, T x L x H dictionary calibrated on the conditional
    branch, CFG batch 2 sharing every cell plan: keep counts = per-(t, l) direct calls
    bitwise; plan = oracle compile; eager step = graph replay = direct per-layer calls bitwise;
    sampled rows of every (t, l) against the fp64 oracle."""
    from paper_2603_05503_b200 import pipeline

    lay, H, d, T, L, prompts = Layout(2, 9, 40, 128), 3, 128, 4, 3, 2
    alphas = [2.0, 1.6, 1.1]  # heads 0, 1 peaky (low row similarity), head 2 row-independent

    def qk(p, t, l):
        q, k, _ = inputs.structured_qk(lay, H, d, head_seed=10 * t + l, prompt_seed=p,
                                       alpha=alphas, repetitive=(2,), device="cuda")
        return q, k

    dic = pipeline.calibrate(lay, T, L, H, prompts, qk, pipeline.DISTILLED, gamma=0.95)
    assert abs(dic.eps[0] - 0.863) < 1e-15 and dic.eps == sorted(dic.eps, reverse=True)
    nb = lay.NB
    kind = dic.plan.kind.cpu().numpy()
    sim = dic.similarity.cpu().numpy()
    bits = unpack_bits(dic.plan.mask_bits.cpu().numpy(), nb).reshape(T * L * H, nb, nb)
    for t in range(T):
        for l in range(L):
            keep = u16_zeros(H * nb * nb)
            for p in range(prompts):
                q, k = qk(p, t, l)
                csa.calib_accumulate(lay, q, k, dic.eps[t], keep)
            c0 = dic.cell_base(t, l)
            got = u16_np(dic.keep_count[c0:c0 + H].reshape(-1))
            assert np.array_equal(got, u16_np(keep))
            for h in range(H):
                ref = oracle.compile_cell(got.reshape(H, nb, nb)[h], lay.N, lay.B, lay.F, lay.H,
                                          lay.W, dic.min_count, similarity=sim[c0 + h],
                                          gamma=0.95)
                assert kind[c0 + h] == ref["kind"]
                if ref["kind"] == 0:
                    assert np.array_equal(bits[c0 + h], ref["mask"])
    assert kind.reshape(T, L, H)[:, :, 2].all(), sim  # generated repetitive head: s ~ 1
    assert not kind.all(), sim                       # MASK cells present as well
    bufs = [qkv(2, lay.N, H, d, seed=100 + l, device="cuda") for l in range(L)]
    outs = [torch.empty_like(b[0]) for b in bufs]
    step = pipeline.DenoiseStep(dic, [b[0] for b in bufs], [b[1] for b in bufs],
                                [b[2] for b in bufs], outs)
    for t in range(T):
        step.run(t)
        torch.cuda.synchronize()
        eager = [o.clone() for o in outs]
        for o in outs:
            o.zero_()
        step.replay(t)
        torch.cuda.synchronize()
        for l in range(L):
            assert torch.equal(outs[l], eager[l])
            direct = csa.sparse_attn_fwd(*bufs[l], dic.plan, step.work[t][l],
                                         cell_base=dic.cell_base(t, l))
            assert torch.equal(direct, eager[l])
            c0 = dic.cell_base(t, l)
            for b in range(2):
                for h in range(H):
                    r = (t + l + h) % nb
                    rows = (r * lay.B, min((r + 1) * lay.B, lay.N))
                    ref, _ = oracle_head(lay, *bufs[l], b, h, mask=bits[c0 + h],
                                         rep_k=5 if kind[c0 + h] else None, rows=rows)
                    assert_close(eager[l][b, rows[0]:rows[1], h].double().cpu().numpy(), ref,
                                 f"t{t} l{l} b{b} h{h}")


@pytest.mark.parametrize("lay", [Layout(1, 1, 100, 128, 192), Layout(1, 3, 50, 128, 64),
                                 Layout(1, 1, 100, 128), Layout(1, 2, 65, 128, 112),
                                 Layout(3, 1, 43, 128, 144)])
def test_rect_edge_layouts_calibrate_compile_attend(csa, lay):
    """Degenerate grids: N below one block (N_B = N_Bkv = 1), a key tail of a few tokens, query
    and key grids with different raggedness, one spatial row per frame (anchor k = H = 1).  The
    whole path: calibration (E, selection), compile, attention (MASK + REPETITIVE), vs oracle."""
    heads, d = 2, 128
    q, k, v = qkv(1, lay.N, heads, d, seed=lay.N + lay.Bkv, device="cuda")
    nb, nbk = lay.NB, lay.NBK
    counts = u16_zeros(heads * nb * nbk)
    energy = torch.empty(heads * nb * nbk, dtype=torch.float32, device="cuda")
    csa.calib_accumulate(lay, q, k, 0.8, counts, energy_out=energy)
    torch.cuda.synchronize()
    E = energy.view(heads, nb, nbk).double().cpu().numpy()
    cnt = u16_np(counts).reshape(heads, nb, nbk)
    scale = 1.0 / np.sqrt(d)
    for h in range(heads):
        E_ref = oracle.block_energy(head64(q, 0, h), head64(k, 0, h), scale, lay.B,
                                    block_kv=lay.BK or None)
        assert np.abs(E[h] - E_ref).max() <= 5e-5
        for r in range(nb):
            assert np.array_equal(oracle.select(E[h, r], 0.8), cnt[h, r])
    plan = check_plan_against_oracle(csa, lay, cnt, 1, sim=[0.0, 1.0], anchor_k=1)
    work = csa.build_work_list(plan, 0, heads)
    out = csa.sparse_attn_fwd(q, k, v, plan, work)
    torch.cuda.synchronize()
    mask0 = (cnt[0] >= 1).astype(np.uint8)
    ref0, _ = oracle_head(lay, q, k, v, 0, 0, mask=mask0)
    assert_close(out[0, :, 0].double().cpu().numpy(), ref0, "mask head")
    ref1, _ = oracle_head(lay, q, k, v, 0, 1, rep_k=1)
    assert_close(out[0, :, 1].double().cpu().numpy(), ref1, "anchor head")


@pytest.mark.parametrize("chunks", [1, 2, 0])  # 0: return exchange fused into the epilogue
def test_sharded_denoise_step_nccl_graph(csa, chunks):
    """f4 on the head-sharded runtime through a real NCCL group (one rank here; the exchange,
    chunk overlap and CUDA-graph capture of the NCCL calls are the N-rank code path): the
    sharded step's output equals the single-GPU DenoiseStep's bit for bit, eager and as a
    replayed graph; rank dictionaries from PlanDictionary.shard hold the full dictionary's cells
    bit for bit (P = 2, LPT order); sampled rows against the fp64 oracle."""
    import socket

    import torch.distributed as dist

    from paper_2603_05503_b200 import pipeline

    lay, H, d, T, L, prompts = Layout(2, 9, 40, 128), 4, 128, 2, 2, 2

    def qk(p, t, l):
        q, k, _ = inputs.structured_qk(lay, H, d, head_seed=10 * t + l, prompt_seed=p,
                                       alpha=[2.0, 1.6, 1.1, 1.4], repetitive=(2,), device="cuda")
        return q, k

    dic = pipeline.calibrate(lay, T, L, H, prompts, qk, pipeline.DISTILLED, gamma=0.95)
    bufs = [qkv(2, lay.N, H, d, seed=200 + l, device="cuda") for l in range(L)]
    ref_o = [torch.empty_like(b[0]) for b in bufs]
    single = pipeline.DenoiseStep(dic, [b[0] for b in bufs], [b[1] for b in bufs],
                                  [b[2] for b in bufs], ref_o)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        outs = [torch.empty_like(b[0]) for b in bufs]
        fused = chunks == 0   # the return exchange fused into the epilogue (symmetric memory)
        step = pipeline.ShardedDenoiseStep(dic.shard(1, 0), 1, [b[0] for b in bufs],
                                           [b[1] for b in bufs], [b[2] for b in bufs],
                                           None if fused else outs, chunks=max(chunks, 1),
                                           fused_out=fused)
        outs = step.o
        for t in range(T):
            single.run(t)
            step.run(t)
            torch.cuda.synchronize()
            for l in range(L):
                assert torch.equal(outs[l], ref_o[l]), (t, l)
            eager = [o.clone() for o in outs]
            for o in outs:
                o.zero_()
            step.replay(t)
            torch.cuda.synchronize()
            for l in range(L):
                assert torch.equal(outs[l], eager[l]), (t, l)
    finally:
        dist.destroy_process_group()
    # rank dictionaries of a 2-way split in LPT order: cell-local compile, the same plans
    perm = [0, 3, 1, 2]
    nb = lay.NB
    full_bits = unpack_bits(dic.plan.mask_bits.cpu().numpy(), nb).reshape(T, L, H, nb, nb)
    full_kind = dic.plan.kind.cpu().numpy().reshape(T, L, H)
    for r in range(2):
        part = dic.shard(2, r, perm)
        bits = unpack_bits(part.plan.mask_bits.cpu().numpy(), nb).reshape(T, L, 2, nb, nb)
        kind = part.plan.kind.cpu().numpy().reshape(T, L, 2)
        for j, h in enumerate(perm[2 * r:2 * r + 2]):
            assert np.array_equal(kind[:, :, j], full_kind[:, :, h])
            assert np.array_equal(bits[:, :, j], full_bits[:, :, h])
    kind = full_kind
    for t in range(T):
        single.run(t)
        torch.cuda.synchronize()
        for l in range(L):
            for h in range(H):
                b, r = (t + h) % 2, (l + h) % nb
                rows = (r * lay.B, min((r + 1) * lay.B, lay.N))
                ref, _ = oracle_head(lay, *bufs[l], b, h, mask=full_bits[t, l, h],
                                     rep_k=5 if kind[t, l, h] else None, rows=rows)
                assert_close(ref_o[l][b, rows[0]:rows[1], h].double().cpu().numpy(), ref,
                             f"t{t} l{l} h{h}")


def test_max_block_grid_whole_path(csa):
    """The largest grid the 16-bit skip lists allow: N_B = 2047 blocks (N = 262 016, one frame
    of 2047 x 128 tokens).  Fused calibration + similarity (every row's selection bit-exact on
    the pass's own E, sampled E rows and one cos(f, i) against the oracle), plan compile (the
    MASK cell bit-exact against the oracle compiler), attention on the CSR and the
    intervals-only plan (bitwise equal; sampled rows against the oracle)."""
    lay = Layout(1, 2047, 128, 128)
    assert lay.NB == 2047
    heads, d, kA = 2, 128, 5
    q, k, v = inputs.structured_qk(lay, heads, d, 7, 0, alpha=[1.3, 1.3], repetitive=(1,),
                                   device="cuda")
    nb = lay.NB
    counts = u16_zeros(heads * nb * nb)
    energy = torch.empty(heads * nb * nb, dtype=torch.float32, device="cuda")
    sim = torch.zeros(heads, dtype=torch.float64, device="cuda")
    cos = torch.empty(heads * lay.F * lay.H, dtype=torch.float32, device="cuda")
    csa.calib_accumulate_sim(lay, q, k, 0.9, counts, kA, sim, energy_out=energy, cos_out=cos)
    torch.cuda.synchronize()
    E = energy.view(heads, nb, nb).double().cpu().numpy()
    cnt = u16_np(counts).reshape(heads, nb, nb)
    for h in range(heads):
        for r in range(nb):
            assert np.array_equal(oracle.select(E[h, r], 0.9), cnt[h, r]), (h, r)
    scale = 1.0 / np.sqrt(d)
    qh, kh = head64(q, 0, 0), head64(k, 0, 0)
    for r in (0, nb - 1):
        E_ref = oracle.block_energy(qh, kh, scale, lay.B, block_rows=(r, r + 1))
        assert np.abs(E[0, r] - E_ref[0]).max() <= 5e-5, r
    c_ref = oracle.spatial_cos(lay.F, lay.H, lay.W, qh, kh, scale, kA, 0, 1000)
    assert abs(cos.view(heads, lay.H)[0, 1000].item() - c_ref) <= 2e-5
    s = sim / float(lay.F * lay.H)
    plans = {}
    for csr in (True, False):
        plans[csr] = csa.compile_plan(lay, counts, 1, similarity=s, gamma=0.87, anchor_k=kA,
                                      csr=csr)
        csa.validate_plan(plans[csr])
    p = plans[True]
    ref_cell = oracle.compile_cell(cnt[0], lay.N, lay.B, lay.F, lay.H, lay.W, 1)
    assert np.array_equal(p.blk_row_ptr.cpu().numpy()[:nb + 1], ref_cell["blk_row_ptr"])
    assert np.array_equal(u16_np(p.blk_idx)[:int(p.blk_base[1].item())], ref_cell["blk_idx"])
    outs = [csa.sparse_attn_fwd(q, k, v, plans[c], csa.build_work_list(plans[c], 0, heads))
            for c in (True, False)]
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    kinds = p.kind_host
    mask0 = (cnt[0] >= 1).astype(np.uint8)
    for h, r in ((0, 0), (0, nb // 2), (0, nb - 1), (1, 3)):
        rows = (r * lay.B, min((r + 1) * lay.B, lay.N))
        ref, _ = oracle_head(lay, q, k, v, 0, h, mask=mask0 if not kinds[h] else None,
                             rep_k=kA if kinds[h] else None, rows=rows)
        assert_close(outs[0][0, rows[0]:rows[1], h].double().cpu().numpy(), ref, f"h{h} r{r}")


def _fuzz_cases(n=64, seed=2026):
    """Seeded random attention problems: geometry (ragged N up to 4000), block 64 / 128, B_kv,
    head_dim, heads, batch, mask density, an anchor head, CSR or intervals-only plan."""
    rng = np.random.default_rng(seed)
    cases = []
    while len(cases) < n:
        B = int(rng.choice([64, 128]))
        BK = 0
        if B == 128 and rng.random() < 0.4:
            BK = int(rng.choice([64, 80, 96, 112, 144, 160, 176, 192]))
        lay = Layout(int(rng.integers(1, 4)), int(rng.integers(1, 10)), int(rng.integers(5, 140)),
                     B, BK)
        if lay.N > 4000:
            continue
        heads = int(rng.integers(1, 4))
        cases.append(dict(lay=lay, d=int(rng.choice([64, 128])), heads=heads,
                          batch=int(rng.integers(1, 3)), dens=float(rng.uniform(0.03, 1.0)),
                          rep=heads >= 2 and rng.random() < 0.5, csr=bool(rng.random() < 0.5),
                          kA=int(rng.integers(1, lay.H + 1)), seed=int(rng.integers(1 << 20))))
    return cases


_FUZZ = _fuzz_cases()


@pytest.mark.parametrize("case", range(len(_FUZZ)))
def test_attention_fuzz_against_oracle(csa, case):
    """Seeded random problems through compile + attention on every kernel (attn.cu at block 64,
    attn5.cu, attn_rect.cu), every output row and LSE of every (batch, head) against the fp64
    oracle on the plan's effective masks (rows emptied by a sparse random mask are repaired by
    the compiler, reading Q7)."""
    c = _FUZZ[case]
    lay, d, heads, batch = c["lay"], c["d"], c["heads"], c["batch"]
    q, k, v = qkv(batch, lay.N, heads, d, seed=c["seed"] % 997, device="cuda")
    rng = np.random.default_rng(c["seed"])
    masks = (rng.random((heads, lay.NB, lay.NBK)) < c["dens"]).astype(np.uint8)
    reps = [heads - 1] if c["rep"] else []
    plan = _plan_from_masks(csa, lay, masks, reps, c["kA"], c["csr"])
    csa.validate_plan(plan)
    bits = unpack_bits(plan.mask_bits.cpu().numpy(), lay.NBK).reshape(heads, lay.NB, lay.NBK)
    lse = torch.empty(batch * heads * lay.N, dtype=torch.float32, device="cuda")
    out = csa.sparse_attn_fwd(q, k, v, plan, csa.build_work_list(plan, 0, heads), lse_out=lse)
    torch.cuda.synchronize()
    lse = lse.view(batch, heads, lay.N).cpu().numpy()
    for b in range(batch):
        for h in range(heads):
            rep = h in reps
            ref, ref_lse = oracle_head(lay, q, k, v, b, h, mask=None if rep else bits[h],
                                       rep_k=c["kA"] if rep else None)
            assert_close(out[b, :, h].double().cpu().numpy(), ref, f"{c} b{b} h{h}")
            assert np.abs(lse[b, h] - ref_lse).max() <= 1e-3, (c, b, h)



def _calib_fuzz_cases(n=16, seed=77):
    rng = np.random.default_rng(seed)
    cases = []
    while len(cases) < n:
        B = int(rng.choice([64, 128, 128]))
        BK = 0
        if B == 128 and rng.random() < 0.25:
            BK = int(rng.choice([64, 80, 144, 192]))
        lay = Layout(int(rng.integers(1, 4)), int(rng.integers(1, 8)), int(rng.integers(5, 120)),
                     B, BK)
        if lay.N > 2000:
            continue
        d = 128 if BK else int(rng.choice([64, 128]))
        cases.append(dict(lay=lay, d=d, heads=int(rng.integers(1, 3)),
                          eps=float(rng.uniform(0.5, 0.99)), kA=int(rng.integers(1, lay.H + 1)),
                          alpha=float(rng.uniform(0.6, 1.6)), seed=int(rng.integers(1 << 20))))
    return cases


_CFUZZ = _calib_fuzz_cases()


@pytest.mark.parametrize("case", range(len(_CFUZZ)))
def test_calib_sim_fuzz_against_oracle(csa, case):
    """Seeded random problems through csa_calib_accumulate_sim (the fused kernel at block 128 x
    128, the two calls' kernels otherwise): E within 5e-5 of the oracle, every row's selection
    bit-exact on the pass's own E, every cos(f, i) within 2e-5."""
    c = _CFUZZ[case]
    lay, d, heads, kA = c["lay"], c["d"], c["heads"], c["kA"]
    q, k, _ = inputs.structured_qk(lay, heads, d, c["seed"] % 101, 0, alpha=[c["alpha"]] * heads,
                                   repetitive=(), device="cuda")
    nb, nbk = lay.NB, lay.NBK
    cnt = u16_zeros(heads * nb * nbk)
    E_t = torch.empty(heads * nb * nbk, dtype=torch.float32, device="cuda")
    sim = torch.zeros(heads, dtype=torch.float64, device="cuda")
    cos_t = torch.empty(heads * lay.F * lay.H, dtype=torch.float32, device="cuda")
    csa.calib_accumulate_sim(lay, q, k, c["eps"], cnt, kA, sim, energy_out=E_t, cos_out=cos_t)
    torch.cuda.synchronize()
    E = E_t.view(heads, nb, nbk).double().cpu().numpy()
    counts = u16_np(cnt).reshape(heads, nb, nbk)
    cos = cos_t.view(heads, lay.F, lay.H).double().cpu().numpy()
    scale = 1.0 / np.sqrt(d)
    for h in range(heads):
        qh, kh = head64(q, 0, h), head64(k, 0, h)
        E_ref = oracle.block_energy(qh, kh, scale, lay.B, block_kv=lay.BK or None)
        assert np.abs(E[h] - E_ref).max() <= 5e-5, (c, h)
        for r in range(nb):
            assert np.array_equal(oracle.select(E[h, r], c["eps"]), counts[h, r]), (c, h, r)
        ref = np.array([[oracle.spatial_cos(lay.F, lay.H, lay.W, qh, kh, scale, kA, f, i)
                         for i in range(lay.H)] for f in range(lay.F)])
        assert np.abs(cos[h] - ref).max() <= 2e-5, (c, h)



def test_head_sharded_calibration_equals_the_dictionary_shard(csa):
    """pipeline.calibrate(heads=...) on each rank's heads (no collective) gives the same keep
    counts, similarity and compiled plans as the full dictionary's shard, bit for bit."""
    from paper_2603_05503_b200 import pipeline
    lay = Layout(2, 9, 40, 128)
    T, L, H, d, prompts = 2, 2, 4, 128, 2

    def qk(p, t, l):
        q, k, _ = inputs.structured_qk(lay, H, d, head_seed=10 * t + l, prompt_seed=p,
                                       alpha=[2.0, 1.6, 1.1, 1.4], repetitive=(2,), device="cuda")
        return q, k

    full = pipeline.calibrate(lay, T, L, H, prompts, qk, pipeline.DISTILLED, gamma=0.95)
    perm = [0, 3, 1, 2]
    for r in range(2):
        mine = perm[2 * r:2 * r + 2]
        part = pipeline.calibrate(lay, T, L, H, prompts, qk, pipeline.DISTILLED, gamma=0.95,
                                  heads=mine)
        ref = full.shard(2, r, perm)
        torch.cuda.synchronize()
        assert torch.equal(part.keep_count.view(torch.int16), ref.keep_count.view(torch.int16))
        assert torch.equal(part.similarity, ref.similarity)
        for name in ("kind", "anchor_k", "mask_bits", "blk_row_ptr", "blk_idx", "ivl", "kept_area"):
            a, b = getattr(part.plan, name), getattr(ref.plan, name)
            if a.dtype == torch.uint16:
                a, b = a.view(torch.int16), b.view(torch.int16)
            assert torch.equal(a, b), (r, name)

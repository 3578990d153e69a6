"""The BRGEMM TPP itself on tcgen05 (K11, brgemm_grouped.cu) through the
reference API: brgemm() / gemm() / matmul() with BF16 inputs under
Engine.AUTO / TENSOR for all three addressing variants, and brgemm_grouped()
(many C blocks per launch).  Tolerance: normwise <= 2e-2 of the reference
(north_star BF16 rule; the tensor core sums a tile's whole batch in one FP32
accumulator, the reference sums per entry then across entries,
contraction.py:295-315).  Every test asserts via tpp_last_config() that the
tensor-core kernel ran."""

import numpy as np
import pytest
import torch

from oracle import tpp_oracle as O

from gpu_util import bf16_bits_to_f32, normwise, to_dev, to_host, vnni_weights

pytestmark = pytest.mark.gpu
tpp = pytest.importorskip("paper_2104_05755_b200")
from paper_2104_05755_b200 import _lib  # noqa: E402

TOL = 2e-2
GROUPED = "brgemm_grouped_kernel<"


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield
    torch.cuda.synchronize()


def _batch(variant, abuf, bbuf, sa, sb, cnt, a0=0, b0=0):
    if variant == "stride":
        return tpp.BrgemmBatch.stride((abuf, a0), (bbuf, b0), sa, sb, cnt)
    if variant == "offset":
        return tpp.BrgemmBatch.offset(abuf, bbuf, [a0 + j * sa for j in range(cnt)], [b0 + j * sb for j in range(cnt)])
    return tpp.BrgemmBatch.address([(abuf, a0 + j * sa) for j in range(cnt)], [(bbuf, b0 + j * sb) for j in range(cnt)])


@pytest.mark.parametrize("variant", ["stride", "offset", "address"])
def test_golden_bf16_cases_on_tensor_cores(golden, variant):
    """The reference-generated BF16 cases (odd shapes, lds, VNNI tails, every
    beta): the tensor engine's element-wise staging path."""
    g = golden("brgemm_cases.npz")
    ran = 0
    for i in range(int(g["count"])):
        key = f"case{i:03d}"
        if str(g[key + "_dtype"]) != "bf16":
            continue
        m, n, k, lda, ldb, ldc, cnt, sa, sb, vnni = (int(v) for v in g[key + "_meta"])
        abuf, bbuf = to_dev(g[key + "_a"]), to_dev(g[key + "_b"])
        c = tpp.TensorView(tpp.TensorDesc(m, n, ldc, tpp.DType.FP32), to_dev(g[key + "_c0"]))
        eng = tpp.Engine.TENSOR if cnt > 0 else tpp.Engine.AUTO   # an empty batch has no GEMM
        spec = tpp.GemmSpec(m, n, k, lda, ldb, ldc, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                            beta=float(g[key + "_beta"]), engine=eng,
                            a_layout=tpp.ALayout.VNNI if vnni else tpp.ALayout.PLAIN)
        tpp.brgemm(spec, _batch(variant, abuf, bbuf, sa, sb, cnt), c)
        got = to_host(c.primary).reshape(-1, ldc)[:n, :m]
        want = g[key + "_c"].reshape(-1, ldc)[:n, :m]
        if cnt > 0:
            assert _lib.last_config().startswith(GROUPED), _lib.last_config()
            ran += 1
        assert normwise(got, want) <= TOL, (i, variant)
    assert ran >= 8


def test_conv_offset_fixture_grouped_and_single(golden):
    """The reference's offset-BRGEMM 3x3 conv fixture (tests/golden/conv.npz,
    made by the unmodified reference): every output row one OFFSET batch of
    R*S*Cb taps -- as single brgemm() calls and as ONE grouped launch."""
    g = golden("conv.npz")
    x, wv, want = g["x"], g["w"], g["out"]
    N, Cb, H, W, bc = x.shape
    Kb, _, R, S, _, bk, _ = wv.shape
    Hp, Wp = H + 2, W + 2
    xp = np.zeros((N, Cb, Hp, Wp, bc), np.uint16)
    xp[:, :, 1:-1, 1:-1] = x
    xd, wd = to_dev(xp), to_dev(wv)
    spec = tpp.GemmSpec(bk, W, bc, bk, bc, bk, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                        a_layout=tpp.ALayout.VNNI, engine=tpp.Engine.TENSOR)
    a_rows, b_rows, c_offs = [], [], []
    out = torch.zeros(N * Kb * H * W * bk, dtype=torch.float32, device="cuda")
    single = torch.zeros_like(out)
    for n in range(N):
        for kb in range(Kb):
            for oh in range(H):
                ao = [(((kb * Cb + cb) * R + r) * S + s) * bc * bk for r in range(R) for s in range(S) for cb in range(Cb)]
                bo = [(((n * Cb + cb) * Hp + oh + r) * Wp + s) * bc for r in range(R) for s in range(S) for cb in range(Cb)]
                co = ((n * Kb + kb) * H + oh) * W * bk
                a_rows.append(ao)
                b_rows.append(bo)
                c_offs.append(co)
                cv = tpp.TensorView(tpp.TensorDesc(bk, W, bk, tpp.DType.FP32), single[co:])
                tpp.brgemm(spec, tpp.BrgemmBatch.offset(wd, xd, ao, bo), cv)
                assert _lib.last_config().startswith(GROUPED)
    tpp.brgemm_grouped(spec, tpp.GroupedBatch.offset(wd, xd, a_rows, b_rows), out, c_offs)
    cfg = _lib.last_config()   # output rows (n, oh) x channel blocks: pairs of kb per tile (gangs)
    assert cfg.startswith(GROUPED) and (f"tiles={N * Kb * H}" in cfg or "gang=2x1" in cfg), cfg
    for res in (out, single):
        got = to_host(res).reshape(N, Kb, H, W, bk)
        assert normwise(got, O.bf16_to_fp32(want)) <= TOL
        assert np.mean(O.fp32_to_bf16_rne(got) == want) > 0.95
    assert torch.equal(out, single)   # same kernel, same per-tile order


@pytest.mark.parametrize("variant", ["stride", "offset", "address", "address_two_buffers"])
def test_cfg2_composition_grouped(variant):
    """BASELINE cfg 2 composed from the BRGEMM TPP the way the reference's
    fc_forward does (kernels.py:312-329): 256 C blocks (token block nb x
    feature block kb), each a 16-entry batch of VNNI weight blocks x input
    blocks -- one grouped tcgen05 launch."""
    rng = np.random.default_rng(90)
    Nb, Cb, bn, bc, Kb, bk = 16, 16, 64, 64, 16, 64
    x = O.fp32_to_bf16_rne(rng.normal(0, 1, (Nb, Cb, bn, bc)).astype(np.float32))
    wv = vnni_weights(rng, Kb, Cb, bk, bc, 0.05)
    xd, wd = to_dev(x), to_dev(wv)
    blk = bc * bk
    spec = tpp.GemmSpec(bk, bn, bc, bk, bc, bk, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                        a_layout=tpp.ALayout.VNNI)
    groups = [(nb, kb) for nb in range(Nb) for kb in range(Kb)]
    if variant == "stride":
        gb = tpp.GroupedBatch.stride(wd, xd, blk, blk, Cb, [kb * Cb * blk for _, kb in groups],
                                     [nb * Cb * blk for nb, _ in groups])
    elif variant == "offset":
        gb = tpp.GroupedBatch.offset(wd, xd, [[(kb * Cb + i) * blk for i in range(Cb)] for _, kb in groups],
                                     [[(nb * Cb + i) * blk for i in range(Cb)] for nb, _ in groups])
    elif variant == "address":
        gb = tpp.GroupedBatch.address([[(wd, (kb * Cb + i) * blk) for i in range(Cb)] for _, kb in groups],
                                      [[(xd, (nb * Cb + i) * blk) for i in range(Cb)] for nb, _ in groups])
    else:   # B blocks from two buffers: raw pointers (cp.async staging)
        xd2 = xd.clone()
        gb = tpp.GroupedBatch.address([[(wd, (kb * Cb + i) * blk) for i in range(Cb)] for _, kb in groups],
                                      [[(xd2 if (nb + i) % 2 else xd, (nb * Cb + i) * blk) for i in range(Cb)]
                                       for nb, _ in groups])
    out = torch.empty(Nb * Kb * bn * bk, dtype=torch.float32, device="cuda")
    tpp.brgemm_grouped(spec, gb, out, [(nb * Kb + kb) * bn * bk for nb, kb in groups])
    # the groups form a full cross product (weight block rows x token blocks):
    # pairs of weight block rows tile together (M = 128 MMAs)
    cfg = _lib.last_config()
    assert cfg.startswith(GROUPED) and "gang=2x1" in cfg, cfg
    # VNNI A through tensor memory, TMA staging (ADDRESS blocks all in one
    # buffer per operand run as offsets from it)
    assert " tmem_a" in cfg and (" tma" in cfg) == (variant != "address_two_buffers"), cfg
    sel = [0, 7, 15]
    _, _, want = O.fc_forward_bf16(x, wv, None, activation=None, nb_sel=sel)   # FP32 pre-narrow
    got = to_host(out).reshape(Nb, Kb, bn, bk)[sel]
    assert normwise(got, want) <= TOL


@pytest.mark.parametrize("variant", ["stride", "offset"])
def test_gangs_partial_and_wide(variant):
    """Gangs of 2 x 4 groups (M = 128 x N = 256 tiles) with partial gangs at
    both edges (11 weight block rows, 121 token blocks): every C block against
    the oracle composition."""
    rng = np.random.default_rng(92)
    Nb, Cb, bn, bc, Kb, bk = 121, 2, 64, 64, 11, 64
    x = O.fp32_to_bf16_rne(rng.normal(0, 1, (Nb, Cb, bn, bc)).astype(np.float32))
    wv = vnni_weights(rng, Kb, Cb, bk, bc, 0.05)
    xd, wd = to_dev(x), to_dev(wv)
    blk = bc * bk
    spec = tpp.GemmSpec(bk, bn, bc, bk, bc, bk, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                        a_layout=tpp.ALayout.VNNI)
    groups = [(nb, kb) for nb in range(Nb) for kb in range(Kb)]
    if variant == "stride":
        gb = tpp.GroupedBatch.stride(wd, xd, blk, blk, Cb, [kb * Cb * blk for _, kb in groups],
                                     [nb * Cb * blk for nb, _ in groups])
    else:
        gb = tpp.GroupedBatch.offset(wd, xd, [[(kb * Cb + i) * blk for i in range(Cb)] for _, kb in groups],
                                     [[(nb * Cb + i) * blk for i in range(Cb)] for nb, _ in groups])
    out = torch.full((Nb * Kb * bn * bk,), float("nan"), dtype=torch.float32, device="cuda")
    tpp.brgemm_grouped(spec, gb, out, [(nb * Kb + kb) * bn * bk for nb, kb in groups])
    assert "gang=2x4" in _lib.last_config(), _lib.last_config()
    sel = [0, 1, 59, 118, 119, 120]          # incl. the last (partial) gang column
    _, _, want = O.fc_forward_bf16(x, wv, None, activation=None, nb_sel=sel)
    got = to_host(out).reshape(Nb, Kb, bn, bk)[sel]
    assert not np.isnan(got).any()
    assert normwise(got, want) <= TOL
    # every block written (the partial gang row / column too)
    assert not torch.isnan(out).any()


@pytest.mark.parametrize("case", ["gang_partial", "m128", "plain", "misaligned_stages"])
def test_tma_staging_modes(case):
    """The TMA staging paths of the grouped kernel against the oracle:
    a partial gang (an empty A sub-block) with VNNI A in tensor memory, one
    M = 128 VNNI block per group (TMEM A, one sub-block), PLAIN A boxes, and
    an OFFSET batch whose blocks start off a row of the TMA views in some
    entries (those stages are staged element-wise by their producer warp)
    while B blocks start mid-row (64-element chunk coordinates, ldb = 256)."""
    rng = np.random.default_rng(93)
    vnni = case != "plain"
    m = 128 if case in ("m128", "plain") else 64
    n, k, ldb = 64, 128, (256 if case == "misaligned_stages" else 128)
    groups, cnt = (5, 3) if case == "gang_partial" else (6, 4)
    lda = m
    ablk = k * m                       # VNNI [k/2][m][2] or PLAIN [k][lda]
    bblk = ldb * n
    a = O.fp32_to_bf16_rne(rng.standard_normal(ablk * (groups * cnt + 2) + 256).astype(np.float32))
    b = O.fp32_to_bf16_rne(rng.standard_normal(bblk * (groups * cnt + 2) + 256).astype(np.float32))
    spec = tpp.GemmSpec(m, n, k, lda, ldb, m, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                        a_layout=tpp.ALayout.VNNI if vnni else tpp.ALayout.PLAIN)
    ad, bd = to_dev(a), to_dev(b)
    rng2 = np.random.default_rng(94)
    if case == "gang_partial":
        # weight block rows kb x token blocks nb (a 5 x 1 cross product of A / B lists -> 3 gangs, the last partial)
        a_lists = [[(g * cnt + i) * ablk for i in range(cnt)] for g in range(groups)]
        b_lists = [[i * bblk for i in range(cnt)] for _ in range(groups)]
    else:
        a_lists = [[int(rng2.integers(0, groups * cnt)) * ablk for _ in range(cnt)] for _ in range(groups)]
        b_lists = [[int(rng2.integers(0, groups * cnt)) * bblk for _ in range(cnt)] for _ in range(groups)]
        if case == "misaligned_stages":
            a_lists[1][2] += 2          # off the 2m-element rows of the A view
            b_lists[3][0] += 64         # mid-row B block: chunk coordinate 1
            b_lists[4][1] += 70         # off any 64-element chunk
    gb = tpp.GroupedBatch.offset(ad, bd, a_lists, b_lists)
    out = torch.full((groups * m * n,), float("nan"), dtype=torch.float32, device="cuda")
    tpp.brgemm_grouped(spec, gb, out, [g * m * n for g in range(groups)])
    cfg = _lib.last_config()
    assert cfg.startswith(GROUPED) and " tma" in cfg, cfg
    if vnni and case != "misaligned_stages":
        assert " tmem_a" in cfg, cfg
    if case == "gang_partial":
        assert "gang=2x1" in cfg, cfg
    got = to_host(out).reshape(groups, n, m)
    for g in range(groups):
        ab = [O.load_a(a, off, m, k, lda, "bf16", vnni=vnni) for off in a_lists[g]]
        bb = [O.load_b(b, off, k, n, ldb, "bf16") for off in b_lists[g]]
        want = O.brgemm(ab, bb, np.zeros((m, n), np.float32), 0.0, "bf16")
        assert normwise(got[g].T, want) <= TOL, (case, g)


@pytest.mark.parametrize("beta", [0.0, 1.0, 0.5])
def test_plain_a_multi_tile_vs_fp64(beta):
    """PLAIN (MN-major) A over several 128 x 256 tiles, ragged edges, padded
    lds, 3 entries, 16-byte staging path."""
    rng = np.random.default_rng(91)
    m, n, k, cnt = 200, 300, 136, 3
    lda, ldb, ldc = 208, 144, 200
    sa, sb = lda * k, ldb * n
    a = O.fp32_to_bf16_rne(rng.standard_normal(sa * cnt).astype(np.float32))
    b = O.fp32_to_bf16_rne(rng.standard_normal(sb * cnt).astype(np.float32))
    c0 = rng.standard_normal(ldc * n).astype(np.float32)
    spec = tpp.GemmSpec(m, n, k, lda, ldb, ldc, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32, beta=beta,
                        engine=tpp.Engine.TENSOR)
    c = tpp.TensorView(tpp.TensorDesc(m, n, ldc, tpp.DType.FP32), torch.from_numpy(c0.copy()).cuda())
    tpp.brgemm(spec, tpp.BrgemmBatch.stride(to_dev(a), to_dev(b), sa, sb, cnt), c)
    assert _lib.last_config().startswith("brgemm_grouped_kernel<128,"), _lib.last_config()  # M=128 tiles
    af, bf = O.bf16_to_fp32(a).astype(np.float64), O.bf16_to_fp32(b).astype(np.float64)
    ref = beta * c0.reshape(n, ldc)[:, :m].T.astype(np.float64)
    for i in range(cnt):
        A = af[i * sa:i * sa + lda * k].reshape(k, lda).T[:m]
        B = bf[i * sb:i * sb + ldb * n].reshape(n, ldb).T[:k]
        ref = ref + A @ B
    got = to_host(c.primary).reshape(n, ldc)[:, :m].T
    assert normwise(got, ref) <= 1e-5   # FP32 accumulation of exact BF16 products


def test_misaligned_blocks_generic_staging():
    """Blocks at odd element offsets (not 16-byte aligned) and odd extents:
    per-stage element-wise staging, VNNI and PLAIN A, beta = -2."""
    rng = np.random.default_rng(92)
    for vnni in (False, True):
        m, n, k, cnt = 37, 50, 21, 4
        lda, ldb, ldc = 41, 23, 39
        asz = (-(-k // 2) * m * 2) if vnni else lda * k
        sa, sb = asz + 3, ldb * n + 5
        a = O.fp32_to_bf16_rne(rng.standard_normal(sa * cnt + 3).astype(np.float32))
        b = O.fp32_to_bf16_rne(rng.standard_normal(sb * cnt + 1).astype(np.float32))
        c0 = rng.standard_normal(ldc * n).astype(np.float32)
        spec = tpp.GemmSpec(m, n, k, lda, ldb, ldc, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32, beta=-2.0,
                            a_layout=tpp.ALayout.VNNI if vnni else tpp.ALayout.PLAIN)
        c = tpp.TensorView(tpp.TensorDesc(m, n, ldc, tpp.DType.FP32), torch.from_numpy(c0.copy()).cuda())
        ad, bd = to_dev(a), to_dev(b)
        tpp.brgemm(spec, tpp.BrgemmBatch.address([(ad, 3 + j * sa) for j in range(cnt)],
                                                 [(bd, 1 + j * sb) for j in range(cnt)]), c)
        assert _lib.last_config().startswith(GROUPED)
        ab = [O.load_a(a, 3 + j * sa, m, k, lda, "bf16", vnni=vnni) for j in range(cnt)]
        bb = [O.load_b(b, 1 + j * sb, k, n, ldb, "bf16") for j in range(cnt)]
        want = O.brgemm(ab, bb, c0.reshape(n, ldc)[:, :m].T.copy(), -2.0, "bf16")
        got = to_host(c.primary).reshape(n, ldc)[:, :m].T
        assert normwise(got, want) <= TOL, vnni


def test_gemm_and_matmul_bf16_use_tensor_cores():
    rng = np.random.default_rng(93)
    m, n, k = 96, 80, 64
    a = tpp.from_array(rng.standard_normal((m, k)).astype(np.float32), tpp.DType.BF16)
    b = tpp.from_array(rng.standard_normal((k, n)).astype(np.float32), tpp.DType.BF16)
    c = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
    tpp.matmul(a, b, c)
    assert _lib.last_config().startswith("brgemm_grouped_kernel<128,")
    ref = O.bf16_to_fp32(tpp.bits_of(a)).astype(np.float64) @ O.bf16_to_fp32(tpp.bits_of(b)).astype(np.float64)
    assert normwise(tpp.to_array(c), ref) <= 1e-5
    # ORDERED stays the bitwise reference order
    c2 = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
    tpp.gemm(tpp.GemmSpec(m, n, k, m, k, m, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                          engine=tpp.Engine.ORDERED), a, b, c2)
    want = O.brgemm([O.bf16_to_fp32(tpp.bits_of(a))], [O.bf16_to_fp32(tpp.bits_of(b))],
                    np.zeros((m, n), np.float32), 0.0, "bf16")
    assert tpp.to_array(c2).tobytes() == np.asarray(want, np.float32).tobytes()


def test_grouped_fallback_other_dtypes_matches_single_calls():
    """brgemm_grouped on FP32 runs one ordered brgemm per group: bitwise equal
    to the single calls (the reference order)."""
    rng = np.random.default_rng(94)
    m = n = k = 16
    G, cnt = 5, 3
    a = torch.from_numpy(rng.standard_normal(G * cnt * m * k).astype(np.float32)).cuda()
    b = torch.from_numpy(rng.standard_normal(G * cnt * k * n).astype(np.float32)).cuda()
    spec = tpp.GemmSpec(m, n, k, m, k, m)
    gb = tpp.GroupedBatch.stride(a, b, m * k, k * n, cnt, [g * cnt * m * k for g in range(G)],
                                 [g * cnt * k * n for g in range(G)])
    out = torch.zeros(G * m * n, dtype=torch.float32, device="cuda")
    tpp.brgemm_grouped(spec, gb, out, [g * m * n for g in range(G)])
    for g in range(G):
        c = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
        tpp.brgemm(spec, tpp.BrgemmBatch.stride((a, g * cnt * m * k), (b, g * cnt * k * n), m * k, k * n, cnt), c)
        assert torch.equal(c.primary, out[g * m * n:(g + 1) * m * n])
    with pytest.raises(tpp.TensorError):
        tpp.brgemm_grouped(spec, gb, out, [0] * G)            # C blocks must be distinct
    with pytest.raises(NotImplementedError):
        tpp.brgemm_grouped(tpp.GemmSpec(m, n, k, m, k, m, engine=tpp.Engine.TENSOR), gb, out,
                           [g * m * n for g in range(G)])


@pytest.mark.parametrize("gang", [False, True])
def test_grouped_bf16_output_column_map(gang):
    """tpp_brgemm_grouped_bf16: the BF16 epilogue (RNE with the reference's
    NaN rule) with a column map (period 10, keep 7) gives the same bits as
    the FP32 grouped call narrowed by the oracle's RNE and remapped -- on a
    ganged (2 x 1, TMEM A) and an ungrouped tiling, with NaN / Inf / tie
    inputs in A."""
    import ctypes as C
    rng = np.random.default_rng(95)
    groups, cnt, m, n, k = 6, 3, 64, 40, 64
    blk = m * k
    a = O.fp32_to_bf16_rne(rng.standard_normal(blk * groups * cnt).astype(np.float32))
    a[5] = 0x7FC1            # NaN
    a[blk + 7] = 0x7F80      # +Inf
    b = O.fp32_to_bf16_rne(rng.standard_normal(k * n * cnt).astype(np.float32))
    ad, bd = to_dev(a), to_dev(b)
    spec = tpp.GemmSpec(m, n, k, m, k, m, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                        a_layout=tpp.ALayout.VNNI)
    a_off = torch.tensor([(g * cnt + i) * blk for g in range(groups) for i in range(cnt)], dtype=torch.int64).cuda()
    b_off = torch.tensor([i * k * n for _ in range(groups) for i in range(cnt)], dtype=torch.int64).cuda()
    acc = torch.empty(groups * m * n, dtype=torch.float32, device="cuda")
    lib = _lib.load()
    d = spec.c()
    d.engine = _lib.ENGINE_TENSOR
    c_off = torch.tensor([g * m * n for g in range(groups)], dtype=torch.int64).cuda()
    _lib.check(lib.tpp_brgemm_grouped(C.byref(d), 1, ad.data_ptr(), bd.data_ptr(), 0, 0, a_off.data_ptr(),
                                      b_off.data_ptr(), cnt, acc.data_ptr(), c_off.data_ptr(), groups, None), "fp32")
    per, keep = 10, 7
    ncols = n // per * keep
    out = torch.full((groups * m * ncols,), -1, dtype=torch.int16, device="cuda")
    c16 = torch.tensor([g * m * ncols for g in range(groups)], dtype=torch.int64).cuda()
    table, ng, gm, gn = None, 0, 1, 1
    if gang:   # rows: groups 2j, 2j+1 (distinct A lists); one B list; cells
        ng, gm, gn = groups // 2, 2, 1
        rows = [g for g in range(groups)]
        cols = [2 * j for j in range(ng)]
        cells = [g for g in range(groups)]
        table = torch.tensor(rows + cols + cells, dtype=torch.int32).cuda()
    _lib.check(lib.tpp_brgemm_grouped_bf16(C.byref(d), 1, ad.data_ptr(), bd.data_ptr(), 0, 0, a_off.data_ptr(),
                                           b_off.data_ptr(), cnt, out.data_ptr(), c16.data_ptr(), groups,
                                           table.data_ptr() if table is not None else None, ng, gm, gn, per, keep,
                                           None), "bf16")
    cfg = _lib.last_config()
    assert cfg.startswith(GROUPED) and (("gang=2x1" in cfg and " tmem_a" in cfg) if gang else True), cfg
    want_full = O.fp32_to_bf16_rne(to_host(acc)).reshape(groups, n, m)       # [g][column][row]
    keep_cols = [v for v in range(n) if v % per < keep]
    want = want_full[:, keep_cols, :]
    got = to_host(out).view(np.uint16).reshape(groups, ncols, m)
    assert np.array_equal(got, want)

"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference TPP algorithms on the BRGEMM hot path
(/root/reference/pkg/src/tensorprim, "tensorprim" 0.1.0).  Nothing in the
product package imports this module: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` leg may use it, and only
as the checker.  Every function cites the reference file:line it restates.

Parity of this restatement is PINNED against the reference itself: the golden
fixtures in ``tests/golden/`` were produced by importing the unmodified
reference package in the build container (``tests/golden/make_golden.py``),
and ``tests/test_oracle_golden.py`` checks every function below against them
bit-for-bit.

Arithmetic rules (the reference's, restated):
  * numpy float32/float64 ``+``/``*`` are separately rounded IEEE ops (no FMA
    contraction), so evaluating the same expression in the same order gives
    the same bits;
  * BRGEMM order (contraction.py:295-315): acc = beta-rule(C); for every batch
    entry i: part = +0, then part += a[m,k]*b[k,n] for k ascending; acc += part.
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# precision codecs — dtypes.py:76-110
# ---------------------------------------------------------------------------


def bf16_to_fp32(bits: np.ndarray) -> np.ndarray:
    """dtypes.py:76-79 — append 16 zero bits."""
    bits = np.asarray(bits, dtype=np.uint16)
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def fp32_to_bf16_rne(values: np.ndarray) -> np.ndarray:
    """dtypes.py:82-97 — RNE on the dropped half; NaN truncated, quiet bit
    0x40 forced when the surviving payload is empty."""
    v = np.asarray(values, dtype=np.float32)
    u = v.view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    rounded = ((u + np.uint32(0x7FFF) + lsb) >> np.uint32(16)).astype(np.uint16)
    trunc = (u >> np.uint32(16)).astype(np.uint16)
    nan_fix = np.where((trunc & np.uint16(0x7F)) == 0, trunc | np.uint16(0x40), trunc)
    return np.where(np.isnan(v), nan_fix, rounded).astype(np.uint16)


def round_bf16(values: np.ndarray) -> np.ndarray:
    """FP32 -> BF16 -> FP32 (value actually representable in BF16)."""
    return bf16_to_fp32(fp32_to_bf16_rne(values))


# ---------------------------------------------------------------------------
# VNNI layouts — contraction.py:238-254, ops.py:573-588
# ---------------------------------------------------------------------------


def vnni_pack_a(a: np.ndarray, alpha: int) -> np.ndarray:
    """contraction.py:238-247 — (M,K) -> flat [ceil(K/alpha)][M][alpha]."""
    m, k = a.shape
    groups = -(-k // alpha)
    out = np.zeros((groups, m, alpha), dtype=a.dtype)
    for g in range(groups):
        for r in range(alpha):
            kk = g * alpha + r
            if kk < k:
                out[g, :, r] = a[:, kk]
    return out.reshape(-1)


def vnni_unpack_a(flat: np.ndarray, alpha: int, m: int, k: int) -> np.ndarray:
    """contraction.py:250-254."""
    groups = -(-k // alpha)
    grid = np.asarray(flat)[: groups * m * alpha].reshape(groups, m, alpha)
    return grid.transpose(1, 0, 2).reshape(m, groups * alpha)[:, :k]


def vnni_pack(a: np.ndarray, alpha: int) -> np.ndarray:
    """ops.py:573-584 — logical (M,N) -> physical (M*alpha, ceil(N/alpha))
    whose column-major flat order is [N/alpha][M][alpha]."""
    m, n = a.shape
    flat = vnni_pack_a(a, alpha)
    groups = -(-n // alpha)
    return flat.reshape(groups, m * alpha).T


def vnni_unpack(packed: np.ndarray, alpha: int, rows: int, cols: int) -> np.ndarray:
    """ops.py:587-592."""
    flat = np.asarray(packed).T.reshape(-1)
    return vnni_unpack_a(flat, alpha, rows, cols)


def vnni_to_vnnit(packed: np.ndarray, alpha: int, alpha_out: int, rows: int, cols: int):
    """ops.py:556-565 — unpack, transpose, repack."""
    return vnni_pack(vnni_unpack(packed, alpha, rows, cols).T, alpha_out)


# ---------------------------------------------------------------------------
# BRGEMM — contraction.py:175-322
# ---------------------------------------------------------------------------


def strided2d(buf: np.ndarray, off: int, rows: int, cols: int, ld: int) -> np.ndarray:
    """contraction.py:175-181 — column-major (rows x cols) window."""
    need = off + ld * (cols - 1) + rows
    if off < 0 or need > buf.size:
        raise ValueError(f"block exceeds buffer: need {need}, have {buf.size}")
    idx = off + np.arange(rows)[:, None] + ld * np.arange(cols)[None, :]
    return buf[idx]


def widen(a: np.ndarray, in_dtype: str) -> np.ndarray:
    """contraction.py:184-189."""
    if in_dtype == "bf16":
        return bf16_to_fp32(a)
    if in_dtype == "int8":
        return a.astype(np.int32)
    return a


def load_a(buf, off, m, k, lda, in_dtype, vnni=False):
    """contraction.py:192-209 (NATIVE path; EMULATED_SPLIT is bit-identical,
    contraction.py:223-235)."""
    if not vnni:
        return widen(strided2d(buf, off, m, k, lda), in_dtype)
    alpha = 4 if in_dtype == "int8" else 2
    groups = -(-k // alpha)
    if off < 0 or buf.size - off < groups * m * alpha:
        raise ValueError("VNNI block exceeds buffer")
    grid = buf[off:off + groups * m * alpha].reshape(groups, m, alpha)
    logical = grid.transpose(1, 0, 2).reshape(m, groups * alpha)[:, :k]
    return widen(logical, in_dtype)


def load_b(buf, off, k, n, ldb, in_dtype):
    """contraction.py:288-289."""
    return widen(strided2d(buf, off, k, n, ldb), in_dtype)


_ACC = {"fp64": np.float64, "fp32": np.float32, "bf16": np.float32, "int8": np.int32}


def brgemm(a_blocks, b_blocks, c0, beta: float, in_dtype: str = "fp32") -> np.ndarray:
    """contraction.py:261-322 — returns the new C (m x n, accumulator dtype).

    ``a_blocks`` are logical (M,K) widened arrays, ``b_blocks`` (K,N); the
    order is the reference's: beta rule (410-415), then per entry a partial
    from +0 along ascending k (417-423), folded onto acc (424).  numpy's
    int32 arithmetic wraps like the reference's.
    """
    acc_t = _ACC[in_dtype]
    c0 = np.asarray(c0)
    m, n = c0.shape
    if beta == 0.0:
        acc = np.zeros((m, n), dtype=acc_t)
    elif beta == 1.0:
        acc = c0.astype(acc_t, copy=True)
    else:
        acc = c0.astype(acc_t, copy=True) * acc_t(beta)
    with np.errstate(all="ignore"):
        for a, b in zip(a_blocks, b_blocks):
            part = np.zeros((m, n), dtype=acc_t)
            for kk in range(a.shape[1]):
                part += a[:, kk:kk + 1] * b[kk:kk + 1, :]
            acc += part
    return acc


def brgemm_blocked(a_stack: np.ndarray, b_stack: np.ndarray, c0=None, beta=0.0) -> np.ndarray:
    """The same per-element order as :func:`brgemm`, vectorised over many
    independent C blocks (what fc_forward's job loop does one block at a
    time, kernels.py:312-329).

    a_stack: [..., I, M, K] widened A blocks; b_stack: [..., I, K, N].
    Leading dims broadcast against each other.  Returns [..., M, N].
    """
    a_stack = np.asarray(a_stack)
    b_stack = np.asarray(b_stack)
    acc_t = a_stack.dtype.type
    lead = np.broadcast_shapes(a_stack.shape[:-3], b_stack.shape[:-3])
    m, n = a_stack.shape[-2], b_stack.shape[-1]
    if beta == 0.0 or c0 is None:
        acc = np.zeros(lead + (m, n), dtype=acc_t)
    elif beta == 1.0:
        acc = np.array(np.broadcast_to(c0, lead + (m, n)), dtype=acc_t)
    else:
        acc = np.array(np.broadcast_to(c0, lead + (m, n)), dtype=acc_t) * acc_t(beta)
    nb = a_stack.shape[-3]
    with np.errstate(all="ignore"):
        for i in range(nb):
            part = np.zeros(lead + (m, n), dtype=acc_t)
            a_i = a_stack[..., i, :, :]
            b_i = b_stack[..., i, :, :]
            for kk in range(a_stack.shape[-1]):
                part += a_i[..., :, kk:kk + 1] * b_i[..., kk:kk + 1, :]
            acc += part
    return acc


# ---------------------------------------------------------------------------
# bitmask companions — tensor.py:238-261
# ---------------------------------------------------------------------------


def bool_to_mask(b: np.ndarray) -> np.ndarray:
    """tensor.py:246-254 — column-major, LSB-first, columns byte-padded."""
    b = np.asarray(b, dtype=bool)
    rows, cols = b.shape
    bpc = (rows + 7) // 8
    padded = np.zeros((bpc * 8, cols), dtype=np.uint8)
    padded[:rows, :] = b
    return np.packbits(padded, axis=0, bitorder="little").T.reshape(-1).copy()


def mask_to_bool(mask: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """tensor.py:257-261."""
    bpc = (rows + 7) // 8
    m = np.asarray(mask, dtype=np.uint8).reshape(cols, bpc).T
    return np.unpackbits(m, axis=0, bitorder="little")[:rows, :].astype(bool)


# ---------------------------------------------------------------------------
# PRNG / dropout — ops.py:195-236 (PrngState), 416-444 (_prng_fill, _dropout),
# 378-382 (DROPOUT_INV)
# ---------------------------------------------------------------------------

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """ops.py:195-199 (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def prng_seed(seed: int, ncols: int) -> np.ndarray:
    """ops.py:210-221 — returns uint32 [4, ncols] = (x, y, z, w)."""
    base = np.arange(ncols, dtype=np.uint64) ^ np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF)
    a = splitmix64(base)
    b = splitmix64(a)
    st = np.stack([a & np.uint64(0xFFFFFFFF), a >> np.uint64(32),
                   b & np.uint64(0xFFFFFFFF), b >> np.uint64(32)]).astype(np.uint32)
    dead = (st[0] | st[1] | st[2] | st[3]) == 0
    st[3] = np.where(dead, np.uint32(1), st[3])
    return st


def prng_step(st: np.ndarray) -> np.ndarray:
    """ops.py:223-228 — advances st in place, returns the new w words."""
    x = st[0]
    t = x ^ (x << np.uint32(11))
    w = st[3]
    nw = (w ^ (w >> np.uint32(19))) ^ (t ^ (t >> np.uint32(8)))
    st[0], st[1], st[2] = st[1].copy(), st[2].copy(), w.copy()
    st[3] = nw
    return nw


def prng_uniform_block(st: np.ndarray, rows: int) -> np.ndarray:
    """ops.py:230-236 — rows x ncols FP32 in [0, 1); row i from step i+1."""
    out = np.empty((rows, st.shape[1]), dtype=np.float32)
    for i in range(rows):
        w = prng_step(st)
        out[i] = (w >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
    return out


def dropout(x: np.ndarray, st: np.ndarray, p: float):
    """ops.py:430-444 — x already widened to its compute dtype; returns
    (values in the compute dtype, keep bool[rows, cols])."""
    u = prng_uniform_block(st, x.shape[0])
    keep = u >= np.float32(p)
    scale = x.dtype.type(1.0 / (1.0 - p))
    with np.errstate(all="ignore"):
        return np.where(keep, x * scale, x.dtype.type(0)), keep


def dropout_inv(x: np.ndarray, keep: np.ndarray, p: float) -> np.ndarray:
    """ops.py:378-382."""
    scale = x.dtype.type(1.0 / (1.0 - p)) if p < 1.0 else x.dtype.type(0)
    with np.errstate(all="ignore"):
        return np.where(keep, x * scale, x.dtype.type(0))


# ---------------------------------------------------------------------------
# QUANTIZE / DEQUANTIZE — ops.py:447-469
# ---------------------------------------------------------------------------


def quantize(x: np.ndarray, scale=None):
    """ops.py:447-460 — returns (int8 array, scale used)."""
    xd = np.asarray(x, dtype=np.float32).astype(np.float64)
    if scale is None:
        amax = float(np.max(np.abs(xd))) if xd.size else 0.0
        scale = amax / 127.0 if amax > 0 else 1.0
    with np.errstate(all="ignore"):
        q = np.clip(np.rint(xd / scale), -127, 127)
    q = np.where(np.isnan(q), 0.0, q).astype(np.int8)  # float64 NaN -> int8 is 0 on x86
    return q, float(scale)


def dequantize(q: np.ndarray, scale: float) -> np.ndarray:
    """ops.py:463-469."""
    return np.asarray(q).astype(np.float32) * np.float32(scale)


# ---------------------------------------------------------------------------
# elementwise TPPs — ops.py:284-386, 747-816
# ---------------------------------------------------------------------------


def relu(x: np.ndarray) -> np.ndarray:
    """ops.py:364 — np.maximum(x, 0): NaN propagates, -0 -> +0."""
    x = np.asarray(x)
    return np.maximum(x, x.dtype.type(0))


def relu_mask(x: np.ndarray) -> np.ndarray:
    """ops.py:365-366 — mask bit is x > 0."""
    return np.asarray(x) > 0


def relu_inv(dy: np.ndarray, mask_bool: np.ndarray) -> np.ndarray:
    """ops.py:367-369."""
    dy = np.asarray(dy)
    return np.where(mask_bool, dy, dy.dtype.type(0))


def binary(kind: str, a, b):
    """ops.py:777-782 (ADD/SUB/MUL/DIV/MAX/MIN) in the compute dtype."""
    fn = {"add": np.add, "sub": np.subtract, "mul": np.multiply,
          "div": np.true_divide, "max": np.maximum, "min": np.minimum}[kind]
    with np.errstate(all="ignore"):
        return fn(a, b)


def muladd(a, b, c, negate=False):
    """ops.py:812-815 — c + a*b (c - a*b), product rounded first."""
    with np.errstate(all="ignore"):
        prod = a * b
        return c - prod if negate else c + prod


def reduce_rows_sum(x: np.ndarray, squared: bool = False) -> np.ndarray:
    """ops.py:484-522 (ROWS, SUM) — FP32 fold from 0 over ascending columns."""
    x = np.asarray(x, dtype=np.float32)
    if squared:
        x = x * x
    acc = np.zeros(x.shape[0], dtype=np.float32)
    for j in range(x.shape[1]):
        acc = acc + x[:, j]
    return acc


def reduce_cols_sum(x: np.ndarray, squared: bool = False) -> np.ndarray:
    """ops.py:484-522 (COLS, SUM) — fold over ascending rows."""
    x = np.asarray(x, dtype=np.float32)
    if squared:
        x = x * x
    acc = np.zeros(x.shape[1], dtype=np.float32)
    for i in range(x.shape[0]):
        acc = acc + x[i, :]
    return acc


# ---------------------------------------------------------------------------
# polynomial approximations — approx.py:100-218, 267-288
# ---------------------------------------------------------------------------


def _interval_bounds(emin: int, i: int):
    """approx.py:120-124."""
    e = emin + i // 2
    lo = 2.0 ** e if i % 2 == 0 else 1.5 * 2.0 ** e
    hi = 1.5 * 2.0 ** e if i % 2 == 0 else 2.0 ** (e + 1)
    return (0.0 if i == 0 else lo), hi


def _cheb_fit(f, a: float, b: float, n: int = 64) -> np.ndarray:
    """approx.py:127-141 — degree-3 Chebyshev projection on n nodes,
    converted to monomial coefficients c0..c3."""
    k = np.arange(n)
    t = np.cos(np.pi * (k + 0.5) / n)
    x = 0.5 * (b - a) * t + 0.5 * (b + a)
    fx = f(x)
    cs = []
    for j in range(4):
        tj = np.cos(j * np.pi * (k + 0.5) / n)
        cs.append((2.0 - (j == 0)) / n * np.sum(fx * tj))
    poly = np.polynomial.chebyshev.Chebyshev(cs, domain=[a, b]).convert(
        kind=np.polynomial.Polynomial)
    c = np.zeros(4)
    c[:poly.coef.size] = poly.coef
    return c


def fit_minimax_table(f, emin: int):
    """approx.py:144-152 — (coeffs[4,16] float32, base, range_max)."""
    coeffs = np.zeros((4, 16))
    for i in range(16):
        a, b = _interval_bounds(emin, i)
        coeffs[:, i] = _cheb_fit(f, a, b)
    return coeffs.astype(np.float32), (127 + emin) << 1, _interval_bounds(emin, 15)[1]


_erf_scaled = np.vectorize(lambda v: math.erf(v / math.sqrt(2.0)), otypes=[np.float64])
GELU_TABLE = fit_minimax_table(_erf_scaled, emin=-5)   # approx.py:158


def minimax_eval(table, x: np.ndarray) -> np.ndarray:
    """approx.py:161-171 (saturation 1.0)."""
    coeffs, base, range_max = table
    x = np.asarray(x, dtype=np.float32)
    dt = np.float32
    ax = np.abs(x)
    bits = ax.view(np.uint32)
    idx = np.clip((bits >> np.uint32(22)).astype(np.int64) - base, 0, 15)
    c0, c1, c2, c3 = (coeffs[j][idx] for j in range(4))
    with np.errstate(all="ignore"):
        p = ((c3 * ax + c2) * ax + c1) * ax + c0
    p = np.where(ax >= dt(range_max), dt(1.0), p)
    return np.copysign(p, x)


def minimax_grad(table, x: np.ndarray) -> np.ndarray:
    """approx.py:174-183."""
    coeffs, base, range_max = table
    x = np.asarray(x, dtype=np.float32)
    dt = np.float32
    ax = np.abs(x)
    bits = ax.view(np.uint32)
    idx = np.clip((bits >> np.uint32(22)).astype(np.int64) - base, 0, 15)
    c1, c2, c3 = (coeffs[j][idx] for j in (1, 2, 3))
    with np.errstate(all="ignore"):
        g = (dt(3.0) * c3 * ax + dt(2.0) * c2) * ax + c1
    return np.where(ax >= dt(range_max), dt(0.0), g)


def gelu(x: np.ndarray) -> np.ndarray:
    """approx.py:267-276 — (0.5*x) * (1 + h), h from the minimax erf table."""
    x = np.asarray(x, dtype=np.float32)
    h = minimax_eval(GELU_TABLE, x)
    with np.errstate(all="ignore"):
        return np.float32(0.5) * x * (np.float32(1.0) + h)


def gelu_grad(x: np.ndarray) -> np.ndarray:
    """approx.py:279-288."""
    x = np.asarray(x, dtype=np.float32)
    dt = np.float32
    h = minimax_eval(GELU_TABLE, x)
    hp = minimax_grad(GELU_TABLE, x)
    with np.errstate(all="ignore"):
        return dt(0.5) * (dt(1.0) + h) + dt(0.5) * x * hp


EXP_LOG2E = np.uint32(0x3FB8AA3B)   # approx.py:50-53
EXP_C1 = np.uint32(0x3F316F7D)
EXP_C2 = np.uint32(0x3E781EEE)
EXP_C3 = np.uint32(0x3D656460)


def exp_taylor(x: np.ndarray) -> np.ndarray:
    """approx.py:190-218 (FP32 path)."""
    x = np.asarray(x, dtype=np.float32)
    f = lambda u: np.uint32(u).view(np.float32)
    log2e, c1, c2, c3 = f(EXP_LOG2E), f(EXP_C1), f(EXP_C2), f(EXP_C3)
    with np.errstate(all="ignore"):
        r = x * log2e
        n = np.rint(r)
        y = r - n
        q = ((c3 * y + c2) * y + c1) * y + np.float32(1.0)
        ni = np.clip(np.nan_to_num(n, nan=0.0), -126, 127).astype(np.int32)
        pow2 = ((ni + np.int32(127)) << np.int32(23)).view(np.float32)
        out = q * pow2
        out = np.where(x > np.float32(88.0), np.float32(np.inf), out)
        out = np.where(x < np.float32(-87.0), np.float32(0.0), out)
    return out.astype(np.float32)


# ---------------------------------------------------------------------------
# composite kernels — kernels.py
# ---------------------------------------------------------------------------


def layernorm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float):
    """kernels.py:134-176 on a logical (rows=instances, cols=features) array.

    Returns (out_fp32, mean_f64, var_f64).  FP32 ascending sums (155-158),
    float64 per-row glue (162-171) stored as FP32 scale/shift, then
    out = B + (shift + x*scale)*G with each op separately rounded (ops.py:812-815).
    ``g``/``b`` broadcast against x.
    """
    x = np.asarray(x, dtype=np.float32)
    rows, cols = x.shape
    s = reduce_rows_sum(x)
    ss = reduce_rows_sum(x, squared=True)
    mu = s.astype(np.float64) / cols
    var = ss.astype(np.float64) / cols - mu * mu
    rstd = 1.0 / np.sqrt(var + eps)
    scale = rstd.astype(np.float32)[:, None]
    shift = (-mu * rstd).astype(np.float32)[:, None]
    with np.errstate(all="ignore"):
        inner = shift + x * scale
        out = np.asarray(b, dtype=np.float32) + inner * np.asarray(g, dtype=np.float32)
    return out, mu, var


def softmax_slice(x: np.ndarray) -> np.ndarray:
    """kernels.py:60-99 for one s1 x s3 slice: max-shift, exp_taylor,
    ALL-sum (rows then columns, ascending; ops.py:519-521), reciprocal, mul."""
    x = np.asarray(x, dtype=np.float32)
    mx = np.max(x)
    with np.errstate(all="ignore"):
        e = exp_taylor(x - mx)
        per_col = reduce_cols_sum(e)
        tot = np.float32(0)
        for v in per_col:
            tot = np.float32(tot + v)
        r = np.float32(1) / tot
        return e * r


def split_sgd_step(w: np.ndarray, grad: np.ndarray, lr: float) -> np.ndarray:
    """kernels.py:235-251 — bitwise FP32 SGD: W - g*fp32(lr) (NMULADD)."""
    with np.errstate(all="ignore"):
        return np.asarray(w, np.float32) - np.asarray(grad, np.float32) * np.float32(lr)


# ---------------------------------------------------------------------------
# blocked FC / conv drivers (compositions of the public reference functions)
# ---------------------------------------------------------------------------


def fc_forward_fp32(a4: np.ndarray, b4: np.ndarray, activation=None) -> np.ndarray:
    """kernels.py:300-329: A[Mb][Kb][bk][bm] x B[Nb][Kb][bn][bk] ->
    C[Nb][Mb][bn][bm] (FP32, beta=0), activation applied per block."""
    a4 = np.asarray(a4, np.float32)
    b4 = np.asarray(b4, np.float32)
    # logical A block (bm x bk) = a4[mb,kb].T ; logical B block (bk x bn) = b4[nb,kb].T
    a_l = a4.transpose(0, 1, 3, 2)[None]            # [1, Mb, Kb, bm, bk]
    b_l = b4.transpose(0, 1, 3, 2)[:, None]         # [Nb, 1, Kb, bk, bn]
    c = brgemm_blocked(a_l, b_l)                    # [Nb, Mb, bm, bn]
    if activation == "relu":
        c = relu(c)
    elif activation == "gelu":
        c = gelu(c)
    return c.transpose(0, 1, 3, 2)                  # [Nb][Mb][bn][bm]


def fc_forward_bf16(x_bits, w_vnni_bits, bias_bits=None, activation=None,
                    residual_bits=None, nb_sel=None):
    """BF16 blocked FC as the reference composition:
    per output block brgemm(BF16, VNNI A, FP32 acc, beta=0) (contraction.py:261),
    + bias (apply_binary ADD, COL broadcast, ops.py:747-782), activation
    (ops.py:361-366), + residual (apply_binary ADD), then convert to BF16 RNE
    (tensor.py:328-355).

    x_bits:      [Nb][Cb][bn][bc]        uint16
    w_vnni_bits: [Kb][Cb][bc/2][bk][2]   uint16
    bias_bits:   [Kb*bk]                 uint16 or None
    residual:    [Nb][Kb][bn][bk]        uint16 or None
    nb_sel:      optional list of token-block indices to compute (subset)
    Returns (out_bits [Nb'][Kb][bn][bk] uint16, relu_mask_bool or None, fp32 pre-narrow).
    """
    x_bits = np.asarray(x_bits)
    if nb_sel is not None:
        x_bits = x_bits[list(nb_sel)]
        if residual_bits is not None:
            residual_bits = np.asarray(residual_bits)[list(nb_sel)]
    Nb, Cb, bn, bc = x_bits.shape
    Kb, Cb2, bc2, bk, two = w_vnni_bits.shape
    assert Cb2 == Cb and bc2 * 2 == bc and two == 2
    # logical A block (bk x bc): A[m,k] = W[kb,cb,k//2,m,k%2]
    a_l = bf16_to_fp32(np.asarray(w_vnni_bits).transpose(0, 1, 3, 2, 4).reshape(Kb, Cb, bk, bc))
    b_l = bf16_to_fp32(x_bits.transpose(0, 1, 3, 2))             # [Nb, Cb, bc, bn]
    acc = brgemm_blocked(a_l[None], b_l[:, None])                  # [Nb, Kb, bk, bn]
    c = acc.transpose(0, 1, 3, 2)                                  # [Nb, Kb, bn, bk]
    with np.errstate(all="ignore"):
        if bias_bits is not None:
            c = c + bf16_to_fp32(bias_bits).reshape(1, Kb, 1, bk)
        mask = None
        if activation == "relu":
            mask = relu_mask(c)
            c = relu(c)
        elif activation == "gelu":
            c = gelu(c)
        if residual_bits is not None:
            c = c + bf16_to_fp32(residual_bits)
    return fp32_to_bf16_rne(c), mask, c


def conv2d_fwd_bf16(x_bits, w_vnni_bits, pad: int = 1, n_sel=None, stride: int = 1):
    """Direct 2-D convolution as an OFFSET-addressed BRGEMM over the R*S taps
    (contraction.py:152-160), on an explicitly zero-padded
    input; FP32 accumulation then BF16 RNE.  Per output row the batch entries
    are the taps in (r, s) order with the Cb input-channel blocks inner; with
    a stride the B block of a tap is every stride-th padded column (ldb =
    stride * bc) of padded row oh * stride + r.

    x_bits: [N][Cb][H][W][bc], w_vnni_bits: [Kb][Cb][R][S][bc/2][bk][2].
    Returns out_bits [N'][Kb][P][Q][bk], P = (H + 2 pad - R) // stride + 1.
    """
    x_bits = np.asarray(x_bits)
    if n_sel is not None:
        x_bits = x_bits[list(n_sel)]
    N, Cb, H, W, bc = x_bits.shape
    Kb, Cb2, R, S, bc2, bk, _ = w_vnni_bits.shape
    xp = np.zeros((N, Cb, H + 2 * pad, W + 2 * pad, bc), dtype=np.uint16)
    xp[:, :, pad:pad + H, pad:pad + W] = x_bits
    xf = bf16_to_fp32(xp)
    # logical A (bk x bc) per (kb, cb, r, s)
    a_l = bf16_to_fp32(np.asarray(w_vnni_bits).transpose(0, 1, 2, 3, 5, 4, 6)
                       .reshape(Kb, Cb, R, S, bk, bc))
    OH, OW = (H + 2 * pad - R) // stride + 1, (W + 2 * pad - S) // stride + 1
    out = np.zeros((N, Kb, OH, OW, bk), dtype=np.float32)
    # batch entries ordered (r, s, cb) — every entry: B block = input row slice
    a_stack = np.stack([a_l[:, cb, r, s] for r in range(R) for s in range(S)
                        for cb in range(Cb)], axis=1)        # [Kb, I, bk, bc]
    for oh in range(OH):
        b_stack = np.stack([xf[:, cb, oh * stride + r, s:s + stride * (OW - 1) + 1:stride, :].transpose(0, 2, 1)
                            for r in range(R) for s in range(S) for cb in range(Cb)],
                           axis=1)                             # [N, I, bc, OW]
        acc = brgemm_blocked(a_stack[None], b_stack[:, None])  # [N, Kb, bk, OW]
        out[:, :, oh] = acc.transpose(0, 1, 3, 2)
    return fp32_to_bf16_rne(out), out


def conv2d_bwd_data_fp64(dout_bits, w_vnni_bits, h: int, w: int, pad: int, stride: int):
    """FP64 restatement of the convolution's adjoint (the forward above is
    out[oh][ow] = sum_{r,s} xpad[oh*stride + r][ow*stride + s] W[r][s]):
    dI[h][w] = sum over (r, s, oh, ow) with oh*stride + r - pad = h,
    ow*stride + s - pad = w of dO[oh][ow] W[r][s].  dout_bits
    [N][Kb][P][Q][bk], weights VNNI [Kb][Cb][R][S][bc/2][bk][2]; returns
    [N][Cb][H][W][bc] float64."""
    do = bf16_to_fp32(np.asarray(dout_bits)).astype(np.float64)
    N, Kb, P, Q, bk = do.shape
    wv = np.asarray(w_vnni_bits)
    _, Cb, R, S, bc2, _, _ = wv.shape
    bc = 2 * bc2
    wl = bf16_to_fp32(wv.transpose(0, 1, 2, 3, 5, 4, 6).reshape(Kb, Cb, R, S, bk, bc)).astype(np.float64)
    hp, wpd = h + 2 * pad + stride, w + 2 * pad + stride
    dip = np.zeros((N, Cb, hp, wpd, bc), dtype=np.float64)
    for r in range(R):
        for s in range(S):
            # contribution of tap (r, s): dip[oh*stride + r][ow*stride + s] += dO[oh][ow] . W[r][s]
            t = np.einsum("nkpqa,kcab->ncpqb", do.reshape(N, Kb, P, Q, bk),
                          wl[:, :, r, s])                       # [N, Cb, P, Q, bc]
            dip[:, :, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride] += t
    return dip[:, :, pad:pad + h, pad:pad + w]


def conv_weights_bwd_data(w_vnni_bits):
    """Backward-data weights: flip the taps and swap in/out channels, i.e.
    VNNI_TO_VNNIT per (r,s) block (ops.py:556-565) on a spatial flip.
    [Kb][Cb][R][S][bc/2][bk][2] -> [Cb][Kb][R][S][bk/2][bc][2]."""
    w = np.asarray(w_vnni_bits)
    Kb, Cb, R, S, bc2, bk, _ = w.shape
    bc = bc2 * 2
    out = np.zeros((Cb, Kb, R, S, bk // 2, bc, 2), dtype=np.uint16)
    for kb in range(Kb):
        for cb in range(Cb):
            for r in range(R):
                for s in range(S):
                    logical = w[kb, cb, r, s].transpose(1, 0, 2).reshape(bk, bc)  # (bk x bc)
                    out[cb, kb, R - 1 - r, S - 1 - s] = (
                        vnni_pack_a(logical.T.copy(), 2).reshape(bk // 2, bc, 2))
    return out


# ---------------------------------------------------------------------------
# blocked MLP training step (BASELINE cfg 5) as a composition of the
# reference TPPs: brgemm over 64-wide reduce blocks (contraction.py:261),
# RELU + bitmask / RELU_INV (ops.py:363-369), softmax (kernels.py:84-99),
# split-SGD (kernels.py:235-251).  Logical row-major matrices; BF16 values
# are carried as exactly-representable FP32.
# ---------------------------------------------------------------------------


def blocked_matmul(x: np.ndarray, w: np.ndarray, blk: int = 64) -> np.ndarray:
    """out[t, o] = sum_c x[t, c] * w[o, c] with the BRGEMM order: batch entries
    are the 64-wide blocks of c (ascending), each a partial from +0 along
    ascending c (contraction.py:295-315).  x [T, C], w [O, C] -> [T, O] FP32."""
    x = np.asarray(x, np.float32)
    w = np.asarray(w, np.float32)
    t, c = x.shape
    o = w.shape[0]
    a_stack = w.reshape(o, c // blk, blk).transpose(1, 0, 2)       # [Cb, O, blk]
    b_stack = x.reshape(t, c // blk, blk).transpose(1, 2, 0)       # [Cb, blk, T]
    return brgemm_blocked(a_stack, b_stack).T                       # [T, O]


def mlp_train_step(x_bits, weights32, targets, lr: float, global_batch: int):
    """One step on one shard.  x_bits: [T, d0] uint16; weights32: list of FP32
    [out, in] masters (the BF16 weight used by the GEMMs is the hi half,
    i.e. the truncated value, as in split-SGD); returns (new weights, dW list,
    per-token loss)."""
    nl = len(weights32)
    wb = [bf16_to_fp32((np.asarray(w, np.float32).view(np.uint32) >> 16).astype(np.uint16))
          for w in weights32]
    h = [bf16_to_fp32(x_bits)]
    masks = [None]
    for l in range(nl - 1):
        z = blocked_matmul(h[l], wb[l])
        masks.append(z > 0)
        h.append(round_bf16(relu(z)))
    logits = blocked_matmul(h[nl - 1], wb[nl - 1])
    tcount, ncls = logits.shape
    p = np.stack([softmax_slice(logits[i:i + 1, :])[0] for i in range(tcount)])
    onehot = np.zeros_like(p)
    onehot[np.arange(tcount), targets] = 1.0
    scale = np.float32(1.0 / global_batch)
    with np.errstate(all="ignore"):
        g = round_bf16((p - onehot) * scale)
        loss = -np.log(p[np.arange(tcount), targets])
    dws = [None] * nl
    for l in range(nl - 1, -1, -1):
        dws[l] = blocked_matmul(g.T.copy(), h[l].T.copy())             # [out, in], tokens reduced
        if l > 0:
            dh = blocked_matmul(g, wb[l].T.copy())                       # [T, in]
            g = round_bf16(relu_inv(dh, masks[l]))
    new = [split_sgd_step(weights32[l], dws[l], lr) for l in range(nl)]
    return new, dws, loss


def dilated_conv1d(x, wt, c: int, k: int, s: int, d: int, q: int) -> np.ndarray:
    """1-D dilated convolution forward (kernels.py:350-378): the reference
    runs, per output block, an address-based BRGEMM over the S taps with
    A_s = W^T block s (K x C) and B_s = input columns at pos + s*d (C x bq);
    per output element that is acc = +0; for s: part = +0; for c ascending:
    part += W[s*C + c, k] * x[c, q + s*d]; acc += part (contraction.py:300-315).
    x: [C, W] FP32; wt: [C*S, K] FP32; returns [K, Q] FP32.
    Vectorised over (k, q); every product and sum rounded as FP32."""
    x = np.asarray(x, np.float32)
    wt = np.asarray(wt, np.float32)
    acc = np.zeros((k, q), np.float32)
    for ss in range(s):
        part = np.zeros((k, q), np.float32)
        for cc in range(c):
            prod = (wt[ss * c + cc, :][:, None] * x[cc, ss * d: ss * d + q][None, :]).astype(np.float32)
            part = (part + prod).astype(np.float32)
        acc = (acc + part).astype(np.float32)
    return acc


def conv2d_bwd_weights(x_bits, dout_bits, R: int = 3, S: int = 3, pad: int = 1) -> np.ndarray:
    """Convolution backward-weights (SURVEY §8(f) 1 — the reference has no
    kernel for it; this is the composition of its forward, kernels/PAPER.md:655,
    with the roles of data and output swapped): for every tap,
        dW[kb][cb][r][s][c][k] = sum_{n, p, q} Xpad[n][cb][p+r][q+s][c] * dO[n][kb][p][q][k]
    evaluated in float64 (the GPU accumulates in FP32 in its own order; tests
    compare normwise).  x_bits [N][Cb][H][W][bc], dout_bits [N][Kb][H][W][bk]
    BF16 patterns; returns float64 [Kb][Cb][R][S][bc][bk]."""
    x = bf16_to_fp32(np.asarray(x_bits)).astype(np.float64)
    do = bf16_to_fp32(np.asarray(dout_bits)).astype(np.float64)
    N, Cb, H, W, bc = x.shape
    _, Kb, _, _, bk = do.shape
    xp = np.zeros((N, Cb, H + 2 * pad, W + 2 * pad, bc))
    xp[:, :, pad:pad + H, pad:pad + W] = x
    dw = np.zeros((Kb, Cb, R, S, bc, bk))
    for r in range(R):
        for s in range(S):
            xs = xp[:, :, r:r + H, s:s + W, :]                       # [N, Cb, H, W, bc]
            dw[:, :, r, s] = np.einsum("nchwi,nkhwj->kcij", xs, do, optimize=True)
    return dw

"""GPU parity for the fused batched GCN layer (NEXT-1, PAPER.md Fig.
algo:graph_conv_batched): Y = sum_ch A_ch (X W_ch + 1 bias_ch^T) against the
fp64 oracle O7.

The kernel (csrc/gcn_fused.cu) evaluates the same value through the exact
identity Y = [A_1 X | ... | A_C X | r] . [W_1; ...; W_C; b] (r_ch = rowsum
A_ch; R26) on the tcgen05 tensor cores.  Tolerance,
per element, relative to the oracle's magnitude sum M = sum_ch sum_e |a_e|
(sum_l |x_jl||w_lc| + |b_c|):
  * Z = A_ch X and r in fp32, storage-order FMA over d <= d_max entries:
    <= d_max * 2^-24 relative to sum |a||x|;
  * 3xTF32 products (default): z*w as zh.wh + zh.wl + zl.wh with zh, wh the
    TF32 truncations and zl, wl the remainders (themselves read at TF32
    precision): <= 3 * 2^-20 |z||w|;
  * the tensor core's fp32 accumulation over 3 * ktot products (ktot = the
    GEMM's K: channels * n_x rounded up to 32 per channel, + 32 per 32
    channels of bias), taken at 2^-23 per addition (truncating accumulator).
  => |Y - Y_ref| <= ((d_max + 2) 2^-24 + 3 * 2^-20 + 3 ktot 2^-23) * M.
Reduced-precision modes replace the split term by the input rounding of both
operands: 2 u_in + u_in^2 (TF32 u_in = 2^-10, BF16 2^-8 round-to-nearest,
taken as 2^-7), with ktot accumulations."""
import numpy as np
import pytest
import torch

import oracle
import paper_1903_11409_b200 as bs
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


# every test runs twice: one CTA per 128-row tile (debug bit 1<<23) and CTA
# pairs (debug bit 1<<22: tcgen05 cta_group::2, M = 256, W split across the
# pair; the default for the fp32 layer over >= 4 x 148 row tiles)
@pytest.fixture(scope="module", params=[1 << 23, 1 << 22], ids=["cta1", "cta_pair"])
def h(request):
    assert torch.cuda.is_available()
    hd = bs.Handle(0)
    hd.set_debug(request.param)
    return hd


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def ktot(channels, n_x):
    return channels * ((n_x + 31) // 32 * 32) + (channels + 31) // 32 * 32


def tol(mode, channels, n_x, dmax):
    K = ktot(channels, n_x)
    if mode == "fp32":
        return (dmax + 2) * 2.0 ** -24 + 3 * 2.0 ** -20 + 3 * K * 2.0 ** -23
    u = {"tf32": 2.0 ** -10, "bf16": 2.0 ** -7}[mode]
    return 2 * u + u * u + (dmax + 2) * 2.0 ** -24 + K * 2.0 ** -23


def channels_of(b, channels, rng):
    """Channel 0 = the batch's graphs; further channels = random subsets of its
    entries with fresh values (same nodes, channel-specific adjacency)."""
    rps, cols, vals = [], [], []
    z = 0
    N = b.n_rows
    rows = np.repeat(np.arange(N), np.diff(b.row_ptr))
    for ch in range(channels):
        keep = np.ones(b.n_nnz, bool) if ch == 0 else rng.random(b.n_nnz) < 0.7
        kept = np.nonzero(keep)[0]
        rp = np.zeros(N + 1, np.int64)
        rp[1:] = np.cumsum(np.bincount(rows[kept], minlength=N))
        rps.append((rp + z).astype(np.int32))
        cols.append(b.col[kept])
        vals.append(b.vals[kept] if ch == 0 else rng.standard_normal(kept.size).astype(np.float32))
        z += kept.size
    return np.stack(rps), np.concatenate(cols).astype(np.int32), np.concatenate(vals).astype(np.float32)


def run_case(h, b, channels, n_x, k, rng, mode="fp32", ldx=None, ldy=None, bias=True, sizes=None, row_off=None):
    rps, col, vals = channels_of(b, channels, rng)
    X = rng.standard_normal((b.n_rows, n_x)).astype(np.float32)
    W = (rng.standard_normal((channels, n_x, k)) / np.sqrt(n_x)).astype(np.float32)
    bi = rng.standard_normal((channels, k)).astype(np.float32) if bias else None
    Xd = T(X) if ldx is None else T(np.pad(X, ((0, 0), (0, ldx - n_x))))[:, :n_x]
    Yd = torch.full((b.n_rows, k if ldy is None else ldy), float("nan"), device=DEV)
    Yv = Yd[:, :k]
    ro = T(b.row_off if row_off is None else row_off)
    h.set_gcn_math(mode)
    try:
        h.gcn_layer(ro, None if sizes is None else T(sizes), T(rps), T(col), T(vals), Xd, T(W),
                    None if bi is None else T(bi), Y=Yv)
        Y = Yv.cpu().numpy()
    finally:
        h.set_gcn_math("fp32")
    ref, mag = oracle.gcn_layer(b.row_off, rps, col, vals, X, W,
                                bi if bi is not None else np.zeros((channels, k), np.float32))
    dmax = int(max(np.diff(rp).max() for rp in rps)) if b.n_rows else 0
    err = np.abs(Y.astype(np.float64) - ref)
    t = tol(mode, channels, n_x, dmax)
    assert not np.isnan(Y).any(), "an element of Y was not written"
    assert np.all(err <= t * mag + 1e-30), (mode, float((err / np.maximum(mag, 1e-300)).max()), t)
    if ldy is not None:
        assert np.isnan(Yd[:, k:].cpu().numpy()).all(), "columns past k were written"
    return Y, ref


@pytest.mark.parametrize("cid,channels,n_x", [(1, 1, 8), (2, 3, 48), (2, 4, 64), (4, 2, 64), (3, 2, 32)])
def test_gcn_layer_parity(h, cid, channels, n_x):
    rng = np.random.default_rng(cid * 10 + channels)
    b = synth.config(cid)
    h.set_hints(int(b.sizes.max()), 0)
    run_case(h, b, channels, n_x, b.k, rng)


@pytest.mark.parametrize("k", [1, 16, 33, 64, 100, 128, 200, 512])
@pytest.mark.parametrize("n_x", [1, 31, 50, 64, 130])
def test_gcn_shapes(h, k, n_x):
    """Output widths across the 32/64/128-feature tiles (partial last tiles),
    input widths not a multiple of the 32-column K block."""
    rng = np.random.default_rng(k * 1000 + n_x)
    b = synth.generate(synth.MOL, (20, 60, 0, 0), 40, 8, seed=k + n_x, dense=False)
    h.set_hints(int(b.sizes.max()), 0)
    run_case(h, b, 2, n_x, k, rng)


@pytest.mark.parametrize("mode", ["fp32", "tf32", "bf16"])
def test_gcn_modes(h, mode):
    """Each precision mode within its bound; the reduced ones must differ from
    the fp32 result somewhere (the mode took effect)."""
    rng = np.random.default_rng(7)
    b = synth.generate(synth.MOL, (20, 60, 0, 0), 100, 8, seed=3, dense=False)
    h.set_hints(int(b.sizes.max()), 0)
    Y, _ = run_case(h, b, 3, 64, 64, np.random.default_rng(7), mode=mode)
    if mode != "fp32":
        Y32, _ = run_case(h, b, 3, 64, 64, np.random.default_rng(7))
        assert not np.array_equal(Y.view(np.uint32), Y32.view(np.uint32))


def test_gcn_leading_dimensions_and_no_bias(h):
    """ldx not a multiple of 4 (the packed-X path), ldy > k (columns past k
    untouched), no bias."""
    rng = np.random.default_rng(11)
    b = synth.generate(synth.MOL, (20, 60, 0, 0), 60, 8, seed=4, dense=False)
    h.set_hints(int(b.sizes.max()), 0)
    run_case(h, b, 2, 37, 96, rng, ldx=41, ldy=100, bias=False)
    run_case(h, b, 2, 64, 64, rng, ldx=68, ldy=72)


def test_gcn_large_graphs_and_channels(h):
    """Graphs larger than a tile and than the staged X halo (rows from global
    memory), 33 channels (two bias blocks, structure read from global
    memory), hints too small."""
    rng = np.random.default_rng(12)
    b = synth.generate(synth.MIX, (100, 400, 1, 5), 6, 8, seed=9, dense=False)
    h.set_hints(0, 0)
    run_case(h, b, 2, 40, 72, rng)
    b2 = synth.generate(synth.MOL, (20, 60, 0, 0), 12, 8, seed=10, dense=False)
    h.set_hints(int(b2.sizes.max()), 0)
    run_case(h, b2, 33, 16, 48, rng)


def test_gcn_padded_layout(h):
    """row_off with gaps between graphs (+ sizes): padding rows are not written."""
    rng = np.random.default_rng(13)
    b = synth.generate(synth.MOL, (20, 60, 0, 0), 30, 8, seed=5, dense=False)
    gap = 7
    ro = np.array([int(b.row_off[i]) + gap * i for i in range(b.batch + 1)], dtype=np.int64)
    Np = int(ro[-1])
    n_x, k, channels = 24, 40, 2
    rps_c, col, vals = channels_of(b, channels, rng)
    rps = np.zeros((channels, Np + 1), np.int32)
    for ch in range(channels):
        for i in range(b.batch):
            n = int(b.sizes[i])
            rps[ch, ro[i]:ro[i] + n + 1] = rps_c[ch, b.row_off[i]:b.row_off[i] + n + 1]
            rps[ch, ro[i] + n:ro[i + 1] + 1] = rps_c[ch, b.row_off[i + 1]]
    X = rng.standard_normal((Np, n_x)).astype(np.float32)
    W = (rng.standard_normal((channels, n_x, k)) / 5).astype(np.float32)
    bias = rng.standard_normal((channels, k)).astype(np.float32)
    Yd = torch.full((Np, k), float("nan"), device=DEV)
    h.set_hints(int(b.sizes.max()), 0)
    h.gcn_layer(T(ro), T(b.sizes), T(rps), T(col), T(vals), T(X), T(W), T(bias), Y=Yd)
    Y = Yd.cpu().numpy()
    Xc = np.concatenate([X[ro[i]:ro[i] + b.sizes[i]] for i in range(b.batch)])
    ref, mag = oracle.gcn_layer(b.row_off, rps_c, col, vals, Xc, W, bias)
    dmax = int(max(np.diff(rp).max() for rp in rps_c))
    t = tol("fp32", channels, n_x, dmax)
    for i in range(b.batch):
        n = int(b.sizes[i])
        got = Y[ro[i]:ro[i] + n].astype(np.float64)
        want, m = ref[b.row_off[i]:b.row_off[i + 1]], mag[b.row_off[i]:b.row_off[i + 1]]
        assert np.all(np.abs(got - want) <= t * m + 1e-30)
        assert np.all(np.isnan(Y[ro[i] + n:ro[i + 1]]))


@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_gcn_layer_reduces_to_spmm(h, cid):
    """W = I, no bias, one channel, integer-valued A and X: the layer is exactly
    the batched SpMM of A with X (every Z value is a small integer, exact in
    TF32, so the 3xTF32 GEMM against I is exact)."""
    b = synth.config(cid, int_valued=True)
    k = min(b.k, 128)
    X = np.ascontiguousarray(b.B[:, :k])
    h.set_hints(int(b.sizes.max()), 0)
    Y = h.gcn_layer(T(b.row_off), None, T(b.row_ptr[None]), T(b.col), T(b.vals), T(X),
                    T(np.eye(k, dtype=np.float32)[None])).cpu().numpy()
    C32 = oracle.spmm_f32(k, b.row_off, None, b.row_ptr, b.col, b.vals, X)
    assert np.array_equal(Y, C32)


@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_gcn_accumulate_writes_each_element_once(h, cid):
    """Write-count check (SURVEY §4 tier 4): with W = I, no bias and C channels
    sharing one integer-valued adjacency, the layer is Y = C * (A X) exactly;
    Y starts as NaN, so an element skipped by every tile stays NaN and one
    covered by two tiles would be written twice with the same value only if
    both tiles computed it -- checked by the exact total."""
    channels = 3
    b = synth.config(cid, int_valued=True)
    k = min(b.k, 128)
    X = np.ascontiguousarray(b.B[:, :k])
    rps = np.stack([b.row_ptr] * channels)
    h.set_hints(int(b.sizes.max()), 0)
    Yd = torch.full((b.n_rows, k), float("nan"), device=DEV)
    h.gcn_layer(T(b.row_off), None, T(rps), T(b.col), T(b.vals), T(X),
                T(np.stack([np.eye(k, dtype=np.float32)] * channels)), Y=Yd)
    AX = oracle.spmm_f32(k, b.row_off, None, b.row_ptr, b.col, b.vals, X)
    assert np.array_equal(Yd.cpu().numpy(), channels * AX)


def test_gcn_big_batch_default_policy():
    """The planner's default at a batch large enough for CTA pairs (4096
    molecule-like graphs = ~1280 row tiles >= 4 x 148): the fp32 layer runs on
    tcgen05 cta_group::2, the TF32 layer on single CTAs; both within their
    derived bounds everywhere, every element written once."""
    hd = bs.Handle(0)
    b = synth.generate(synth.MOL, (20, 60, 0, 0), 4096, 8, seed=21, dense=False)
    assert (b.n_rows + 127) // 128 >= 4 * 148
    hd.set_hints(int(b.sizes.max()), 0)
    run_case(hd, b, 2, 64, 256, np.random.default_rng(21))
    run_case(hd, b, 2, 64, 256, np.random.default_rng(22), mode="tf32")

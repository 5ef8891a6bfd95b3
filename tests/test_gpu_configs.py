"""GPU parity at every BASELINE.json configuration, through the kernel variant
the planner actually picks for that shape (asserted with
shflbw_cu_last_plan), against the oracle.

  * compress_shflbw (src/formats.cpp:140-181) at M > 4096 (the planner's
    chunked ranks; beyond M = 28672 the sort-based pipeline): covered by
    test_gpu_parity.py's full-size digest cases (16384 x 4096 V=64, 8192 x
    2048 V=32, 8192 x 1024 V=128, pinned to the compiled reference) plus a
    non-conformant M = 8192 mask, planner-vs-sort-pipeline equality and an M
    = 40960 case here;
  * the large-FFN SpMM (16384 x 4096, N = 8192, 75 %) run at full size with
    the auto plan (persistent kernel), column slices checked against
    oracle.spmm (spmm_execute, src/spmm.cpp:76-146) -- output columns are
    independent, so a slice of B gives that slice of C;
  * a persistent case whose groups are deeper than one column-index window
    (24 K blocks > kMetaBlocks = 16: the window reload);
  * ResNet-50 batch-32 stride-1 convs (conv2d, src/spmm.cpp:193-291) through
    conv_prepare + the auto plan: 3x3 @56/@28/@14/@7 and 1x1 @56/@14, output
    batch slices checked against oracle.conv2d (a batch element's output
    depends only on its own input), the @7 layer also unsplit so one CTA
    walks its 18+ K blocks over several column-index windows;
  * the converter on the reference's acceptance fuzz (criterion 7,
    tests/acceptance.cpp:295-352): the same 10,000 masks from mt19937_64(7007)
    through the GPU validator and converter, bit-exact against the oracle.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def sb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_05016_b200 as sb
    for k in ("force_simt", "split", "stages", "split_mode", "cp_async_slabs", "persistent", "no_bulk_out",
              "gather_warps", "raster", "tile_n"):
        sb.set_option(k, 0)
    sb.set_option("strict", 1)  # a silent CUDA-core fallback would fail these tests
    yield sb
    sb.set_option("strict", 0)


def dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


def tc_plan(sb):
    plan = sb.last_plan()
    assert plan.startswith("k_spmm_tc") or plan.startswith("k_spmm_persist"), plan
    return plan


def plan_field(plan, key):
    for tok in plan.split():
        if tok.startswith(key + "="):
            return tok.split("=", 1)[1]
    return None


# ---------------------------------------------------------------- converter

def test_compress_nonconformant_m8192(sb, oracle):
    """M = 8192 (radix-sort path): one broken support class; the GPU
    validator's fail_row and the converter's NonConformantMask row match the
    oracle (the lexicographically first failing class's smallest row)."""
    M, K, V = 8192, 1024, 32
    mask = oracle.random_shflbw_mask(M, K, V, 256, oracle.rng(77))
    rs = np.random.RandomState(3)
    for _ in range(3):
        mask[rs.randint(M), rs.randint(K)] ^= 1
    want = oracle.validate(mask, V)
    assert not want[0]
    assert sb.validate_pattern(dev(mask), "shfl_bw", V) == (False, want[1])
    with pytest.raises(sb.NonConformantMask, match=rf"\(row {want[1]}\)"):
        sb.compress_shflbw(torch.zeros(M, K, device="cuda"), dev(mask), V)


def _criterion7_masks(oracle, cases=10000):
    """tests/acceptance.cpp:295-317 with the reference's generator stream."""
    rng = oracle.rng(7007)
    for i in range(cases):
        v = 1 + rng() % 4
        m = v * (1 + rng() % 5)
        k = 1 + rng() % 8
        if i % 3 == 0:
            cpg = rng() % (k + 1)
            mask = oracle.random_shflbw_mask(m, k, v, cpg, rng)
        else:
            mask = np.array([rng() % 2 for _ in range(m * k)], np.uint8).reshape(m, k)
        yield v, mask


def test_converter_acceptance_fuzz_10000(sb, oracle):
    """Criterion 7 at the reference's scale: 10,000 fuzzed masks; the GPU
    validator agrees with the oracle's (fail_row included), the GPU converter
    accepts exactly the conformant ones, and every accepted mask packs
    bit-identically (row_indices, group column lists, values)."""
    accepted = 0
    for i, (v, mask) in enumerate(_criterion7_masks(oracle)):
        m, k = mask.shape
        want_pass, want_row = oracle.validate(mask, v)
        got = sb.validate_pattern(dev(mask), "shfl_bw", v)
        assert got == (bool(want_pass), want_row), (i, v, mask.tolist())
        W = oracle.round16(oracle.random_dense(m, k, i))
        if want_pass:
            a = sb.compress_shflbw(dev(W), dev(mask), v)
            p = oracle.compress(W, mask, v)
            ri, gn, cols, vals = a.to_host()
            assert np.array_equal(ri, p.row_indices) and np.array_equal(gn, p.group_ncols), i
            assert np.array_equal(cols, p.cols), i
            assert np.array_equal(vals.view(np.uint32), oracle.round16(p.values).view(np.uint32)), i
            accepted += 1
        else:
            with pytest.raises(sb.NonConformantMask):
                sb.compress_shflbw(dev(W), dev(mask), v)
    assert accepted > 0


# ---------------------------------------------------------------- SpMM at full size

def test_large_ffn_spmm_auto_plan(sb, oracle):
    """16384 x 4096, N = 8192, V = 64, 75 %: the persistent kernel the planner
    picks for the bench's large-FFN layer, fp32 and bf16 output; two 128-column
    slices of C against oracle.spmm on the same slices of B."""
    M, K, N, V = 16384, 4096, 8192, 64
    cpg = 1024
    mask = oracle.random_shflbw_mask(M, K, V, cpg, oracle.rng(1234))
    W = oracle.round16(oracle.random_dense(M, K, 1))
    a = sb.compress_shflbw(dev(W), dev(mask), V)
    p = oracle.compress(W, mask, V)
    del W, mask
    B = oracle.round16(oracle.random_dense(K, N, 2))
    Bd = dev(B, torch.bfloat16)
    C = sb.spmm_execute(a, Bd)
    plan = tc_plan(sb)
    assert plan.startswith("k_spmm_persist"), plan
    C16 = sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16)
    assert sb.last_plan().startswith("k_spmm_persist"), sb.last_plan()  # (stages depend on the output tile)
    for c0 in (0, N - 128):
        want = oracle.spmm(p, np.ascontiguousarray(B[:, c0:c0 + 128]))
        got = C[:, c0:c0 + 128].cpu().numpy()
        assert oracle.rel_frobenius(got, want) <= TOL, (c0, plan)
        assert np.array_equal(C16[:, c0:c0 + 128].float().cpu().numpy(), oracle.round16(got))


def test_persistent_deep_groups_window_reload(sb, oracle):
    """Auto plan = persistent (320 units > one wave), every group 24 K blocks
    deep: the gather warps reload the column-index window mid-unit
    (kMetaBlocks = 16).  Bitwise equal across 4 / 8 gather warps and 1 / 2
    CTAs per SM; a column slice against the oracle."""
    M, K, N, V = 2048, 6144, 1280, 64
    mask = oracle.random_shflbw_mask(M, K, V, K // 4, oracle.rng(1234))
    W = oracle.round16(oracle.random_dense(M, K, 1))
    B = oracle.round16(oracle.random_dense(K, N, 2))
    a = sb.compress_shflbw(dev(W), dev(mask), V)
    p = oracle.compress(W, mask, V)
    Bd = dev(B, torch.bfloat16)
    got = sb.spmm_execute(a, Bd).cpu().numpy()
    plan = tc_plan(sb)
    assert plan.startswith("k_spmm_persist"), plan
    assert a.total_cols // a.group_count() // 64 >= 24
    want = oracle.spmm(p, np.ascontiguousarray(B[:, :256]))
    assert oracle.rel_frobenius(got[:, :256], want) <= TOL
    for gw, per_sm in ((4, 2), (8, 1), (4, 1)):
        sb.set_option("gather_warps", gw)
        sb.set_option("persistent", per_sm)
        other = sb.spmm_execute(a, Bd).cpu().numpy()
        assert np.array_equal(other, got), (gw, per_sm, sb.last_plan())
    sb.set_option("gather_warps", 0)
    sb.set_option("persistent", 0)


@pytest.mark.parametrize("M,N,K,V,alpha", [
    (2048, 128, 2048, 64, 0.25),   # north star
    (2048, 128, 2048, 32, 0.25),
    (2048, 128, 2048, 128, 0.25),
    (512, 512, 512, 32, 0.1),      # Transformer attention projection, 90 %
    (2048, 1024, 512, 64, 0.5),    # FFN1, 50 %
    (512, 4096, 2048, 128, 0.25),  # FFN2, N = 4096
    (4096, 128, 1024, 64, 0.05),   # GNMT, 95 %
    (4096, 128, 1024, 32, 0.5),    # GNMT, 50 %
])
def test_baseline_spmm_configs_auto_plan(sb, oracle, M, N, K, V, alpha):
    """BASELINE.json configs[0..2] shapes through the auto plan (whatever
    split / persistent variant it picks), fp32 out against the oracle and
    bf16 out = the fp32 result rounded once."""
    cpg = int(np.floor(alpha * K + 0.5))
    mask = oracle.random_shflbw_mask(M, K, V, cpg, oracle.rng(1234))
    W = oracle.round16(oracle.random_dense(M, K, 1))
    B = oracle.round16(oracle.random_dense(K, N, 2))
    a = sb.compress_shflbw(dev(W), dev(mask), V)
    p = oracle.compress(W, mask, V)
    Bd = dev(B, torch.bfloat16)
    got = sb.spmm_execute(a, Bd).cpu().numpy()
    plan = tc_plan(sb)
    ref = oracle.spmm(p, B)
    assert oracle.rel_frobenius(got, ref) <= TOL, plan
    got16 = sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(got16, oracle.round16(got)), plan
    # the error against a float64 recomputation separates the CPU
    # fp32 error from the tensor core's; the bf16-out mode is within one bf16
    # ulp of the oracle per element
    c64 = (W.astype(np.float64) * mask) @ B.astype(np.float64)
    e_gpu, e_ref = oracle.rel_frobenius(got, c64), oracle.rel_frobenius(ref, c64)
    print(f"{plan}: rel err vs f64 -- GPU fp32 {e_gpu:.2e}, CPU oracle fp32 {e_ref:.2e}")
    assert e_gpu <= TOL and e_ref <= TOL
    # (elements whose magnitude is far below the typical one are results of
    # cancellation: there the fp32 accumulation-order error of either side
    # exceeds a bf16 ulp of the tiny result, so they are excluded from the
    # per-element check -- the fp32 relative-Frobenius bound above covers them)
    r16 = oracle.round16(ref).astype(np.float64)
    mag = np.maximum(np.abs(r16), np.abs(got16.astype(np.float64)))
    ulp = np.where(mag > 0, 2.0 ** (np.floor(np.log2(np.where(mag > 0, mag, 1.0))) - 7), 0.0)
    ok = np.abs(got16 - r16) <= ulp
    big = np.abs(ref) >= 2.0 ** -6 * np.sqrt(np.mean(ref.astype(np.float64) ** 2))
    print(f"  bf16 out within 1 ulp of the oracle: {ok.mean() * 100:.3f} % of all elements, "
          f"{ok[big].mean() * 100:.3f} % of those >= rms/64")
    assert np.all(ok[big]), plan


# ---------------------------------------------------------------- ResNet-50 convs

RESNET = [  # name, C, H, K_f, R, V
    ("3x3_64@56", 64, 56, 64, 3, 64),
    ("3x3_128@28", 128, 28, 128, 3, 64),
    ("3x3_256@14", 256, 14, 256, 3, 64),
    ("3x3_512@7", 512, 7, 512, 3, 64),
    ("1x1_256to64@56", 256, 56, 64, 1, 64),
    ("1x1_1024to256@14", 1024, 14, 256, 1, 64),
]


@pytest.mark.parametrize("name,C,H,Kf,R,V", RESNET, ids=[r[0] for r in RESNET])
def test_resnet50_b32_conv_auto_plan(sb, oracle, name, C, H, Kf, R, V):
    Nb, pad = 32, (R - 1) // 2
    crs = C * R * R
    mask = oracle.random_shflbw_mask(Kf, crs, V, crs // 4, oracle.rng(5))
    Wt = oracle.round16(oracle.random_dense(Kf, crs, 6))
    x = oracle.round16(oracle.fill_uniform(oracle.rng(7), C * H * H * Nb).reshape(C, H, H, Nb))
    w = sb.compress_shflbw(dev(Wt), dev(mask), V)
    if R > 1:
        w = sb.conv_prepare(w, R)
    xd = dev(x, torch.bfloat16)
    geo = sb.ConvGeometry(R, R, 1, pad)
    got = sb.conv2d(w, xd, geo).cpu().numpy()
    plan = tc_plan(sb)
    assert plan_field(plan, "kind") == ("2" if R > 1 else "0"), plan
    p = oracle.compress(Wt, mask, V)
    outs = {"auto": got}
    if name == "3x3_512@7":
        # one CTA per unit, no K split: a CTA walks every K block of its group
        # (> 16: several column-index windows)
        sb.set_option("split", 1)
        sb.set_option("persistent", -1)
        outs["unsplit"] = sb.conv2d(w, xd, geo).cpu().numpy()
        up = tc_plan(sb)
        assert plan_field(up, "split") == "none" and up.startswith("k_spmm_tc"), up
        assert w.total_cols // w.group_count() // 64 > 16
        sb.set_option("split", 0)
        sb.set_option("persistent", 0)
    for b0 in (0, Nb - 2):  # batch slices: output image b depends only on input image b
        want = oracle.conv2d(p, np.ascontiguousarray(x[:, :, :, b0:b0 + 2]), R, R, 1, pad)
        for k, o in outs.items():
            assert oracle.rel_frobenius(np.ascontiguousarray(o[:, :, :, b0:b0 + 2]), want) <= TOL, (k, plan)


# ------------------------------------------------- converter planner paths

def _packing(a):
    ri, gn, cols, vals = a.to_host()
    gp, ci, vv = a.raw()
    return [ri, gn, cols, vals.view(np.uint32), gp, ci, vv]


@pytest.mark.parametrize("M,K,V,cpg", [(2048, 2048, 64, 512),    # one-CTA planner (CTA sort)
                                       (8192, 1024, 32, 256),    # chunked ranks
                                       (16384, 512, 64, 128),
                                       (32768, 128, 64, 32),     # 32 chunks
                                       (6144, 100, 3, 40),       # V not a power of two, K % 16 != 0
                                       (4096, 64, 1, 20),        # V = 1: G = M
                                       (8192, 64, 1, 20)])
def test_compress_planner_equals_sort_pipeline(sb, oracle, M, K, V, cpg):
    """The class-table planner (default) and the sort-based pipeline
    (option converter_legacy) give bit-identical matrices, equal to the
    oracle (src/formats.cpp:140-181)."""
    mask = oracle.random_shflbw_mask(M, K, V, cpg, oracle.rng(M + K + V))
    W = oracle.round16(oracle.random_dense(M, K, 5))
    a = sb.compress_shflbw(dev(W), dev(mask), V)
    sb.set_option("converter_legacy", 1)
    try:
        b = sb.compress_shflbw(dev(W), dev(mask), V)
    finally:
        sb.set_option("converter_legacy", 0)
    for x, y in zip(_packing(a), _packing(b)):
        assert np.array_equal(x, y)
    p = oracle.compress(W, mask, V)
    ri, gn, cols, vals = a.to_host()
    assert np.array_equal(ri, p.row_indices) and np.array_equal(gn, p.group_ncols)
    assert np.array_equal(cols, p.cols)
    assert np.array_equal(vals.view(np.uint32), oracle.round16(p.values).view(np.uint32))


def test_compress_beyond_planner_m40960(sb, oracle):
    """M = 40960 > the planner's bound (16-bit row ids, 32 chunks): the
    sort-based pipeline, bit-exact against the oracle."""
    M, K, V = 40960, 128, 64
    mask = oracle.random_shflbw_mask(M, K, V, 40, oracle.rng(11))
    W = oracle.round16(oracle.random_dense(M, K, 6))
    a = sb.compress_shflbw(dev(W), dev(mask), V)
    p = oracle.compress(W, mask, V)
    ri, gn, cols, vals = a.to_host()
    assert np.array_equal(ri, p.row_indices) and np.array_equal(gn, p.group_ncols)
    assert np.array_equal(cols, p.cols)
    assert np.array_equal(vals.view(np.uint32), oracle.round16(p.values).view(np.uint32))


@pytest.mark.parametrize("M,K,V", [(2048, 256, 16), (12288, 256, 64)])
def test_planner_nonconformant_both_paths(sb, oracle, M, K, V):
    """A broken class: the planner and the sort pipeline report the oracle's
    fail_row (lexicographically first failing class, smallest row)."""
    mask = oracle.random_shflbw_mask(M, K, V, 60, oracle.rng(3))
    rs = np.random.RandomState(M)
    for _ in range(2):
        mask[rs.randint(M), rs.randint(K)] ^= 1
    want = oracle.validate(mask, V)
    assert not want[0]
    for legacy in (0, 1):
        sb.set_option("converter_legacy", legacy)
        try:
            assert sb.validate_pattern(dev(mask), "shfl_bw", V) == (False, want[1])
            with pytest.raises(sb.NonConformantMask, match=rf"\(row {want[1]}\)"):
                sb.compress_shflbw(torch.zeros(M, K, device="cuda"), dev(mask), V)
        finally:
            sb.set_option("converter_legacy", 0)


@pytest.mark.parametrize("M,K,V", [(2048, 300, 64), (8192, 256, 256), (1024, 64, 16)])
@pytest.mark.parametrize("din", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("dout", ["bf16", "f16", "f32"])
def test_compress_value_dtypes(sb, oracle, M, K, V, din, dout):
    """Every (dense dtype, value dtype) pair through the fused pack kernel (V
    <= 128) and the wide-group pack path (V = 256): values are the dense
    entries converted with round-to-nearest-even, columns and row indices
    bit-exact against the oracle."""
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}
    mask = oracle.random_shflbw_mask(M, K, V, K // 4, oracle.rng(M + V))
    Wf = oracle.random_dense(M, K, 3)
    Wd = torch.from_numpy(Wf).cuda().to(tdt[din])
    a = sb.compress_shflbw(Wd, dev(mask), V, dtype=tdt[dout])
    Win = Wd.float().cpu().numpy()  # what the converter read
    p = oracle.compress(Win, mask, V)
    ri, gn, cols, vals = a.to_host()
    assert np.array_equal(ri, p.row_indices) and np.array_equal(gn, p.group_ncols)
    assert np.array_equal(cols, p.cols)
    want = torch.from_numpy(np.ascontiguousarray(p.values)).to(tdt[dout]).float().numpy()
    assert np.array_equal(vals, want)

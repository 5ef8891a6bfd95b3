"""GPU parity: the sm_100a path (through the C ABI) against the oracle.

Inputs follow SURVEY.md §8(d): synthetic W, B from the reference's own
generators, rounded to bf16 (RNE) before BOTH sides see them, so operands
are identical and every product is exact in fp32.  Bars:
  * converter: bit-exact row permutation, group column lists, padded device
    layout and bf16 values;
  * CUDA-core path (any V): bit-exact vs the reference's pinned order;
  * tcgen05 path: rel. Frobenius error <= 1e-5 vs the fp32 oracle (the
    reference's own --check bar, tools/shflbw.cpp:33) in fp32-output mode,
    and in bf16-output mode exactly that fp32 result rounded once (RNE).
"""
import hashlib

import os

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def sb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_05016_b200 as sb
    for k, v in (("force_simt", 0), ("split", 0), ("stages", 0), ("split_mode", 0), ("cp_async_slabs", 0),
                 ("persistent", 0), ("no_bulk_out", 0),
                 ("gather_warps", int(os.environ.get("SBW_GATHER_WARPS", "0")))):  # env: run the suite at 4 / 8
        sb.set_option(k, v)
    return sb


def dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def synthetic(oracle, M, K, N, V, alpha, seed=1234):
    """SURVEY §8(d) synthetic inputs: mask random_shflbw_mask(..., mt19937_64(1234)),
    W = random_dense(M,K,1), B = random_dense(K,N,2), bf16-rounded."""
    cpg = int(np.floor(alpha * K + 0.5))
    mask = oracle.random_shflbw_mask(M, K, V, cpg, oracle.rng(seed))
    W = oracle.round16(oracle.random_dense(M, K, 1))
    B = oracle.round16(oracle.random_dense(K, N, 2))
    return mask, W, B


def compress_both(sb, oracle, W, mask, V):
    a = sb.compress_shflbw(dev(W), dev(mask), V)
    return a, oracle.compress(W, mask, V)


def assert_same_packing(a, p, oracle):
    ri, gn, cols, vals = a.to_host()
    assert np.array_equal(ri, p.row_indices)
    assert np.array_equal(gn, p.group_ncols)
    assert np.array_equal(cols, p.cols)
    assert np.array_equal(vals.view(np.uint32), oracle.round16(p.values).view(np.uint32))
    gp, ci, vv = a.raw()
    egp, eci, evv = oracle.pack_device(p, 64, "bf16")
    assert np.array_equal(gp, egp)
    assert np.array_equal(ci, eci)
    assert np.array_equal(vv, evv)


# ---------------------------------------------------------------- converter

@pytest.mark.parametrize("case", load_golden("formats_kat.json")["compress"], ids=lambda c: c["name"])
def test_compress_known_answers(sb, oracle, case):
    if case["name"] == "shape_mismatch":
        with pytest.raises(sb.ShapeMismatch):
            sb.compress_shflbw(torch.zeros(2, 2, device="cuda"), torch.zeros(2, 3, dtype=torch.uint8,
                                                                            device="cuda"), 2)
        return
    dense = np.array(case["dense_bits"], np.uint32).view(np.float32).reshape(case["dense_shape"])
    mask = np.array(case["mask"], np.uint8).reshape(case["mask_shape"])
    V = case["V"]
    if case["status"] == 3:
        with pytest.raises(sb.BadParams):
            sb.compress_shflbw(dev(dense), dev(mask), V)
        return
    if case["status"] == 2:
        with pytest.raises(sb.NonConformantMask, match=rf"\(row {case['fail_row']}\)"):
            sb.compress_shflbw(dev(dense), dev(mask), V)
        assert sb.validate_pattern(dev(mask), "shfl_bw", V) == (False, case["fail_row"])
        return
    a = sb.compress_shflbw(dev(dense), dev(mask), V)
    want = case["packed"]
    ri, gn, cols, vals = a.to_host()
    assert ri.tolist() == want["row_indices"]
    assert gn.tolist() == want["group_ncols"]
    assert cols.tolist() == want["cols"]
    wv = oracle.round16(np.array(want["values_bits"], np.uint32).view(np.float32))
    assert np.array_equal(vals, wv)
    d = sb.decompress(a).cpu().numpy()
    assert np.array_equal(d, oracle.round16(
        np.array(case["decompressed_bits"], np.uint32).view(np.float32).reshape(d.shape)))


def test_compress_random_sequences(sb, oracle):
    for case in load_golden("compress_random.json"):
        m, k, V = case["m"], case["k"], case["V"]
        mask = np.array(case["mask"], np.uint8).reshape(m, k)
        if case["suite"] == "roundtrip":
            W = oracle.round16(oracle.random_dense(m, k, case["dense_seed"]))
            a = sb.compress_shflbw(dev(W), dev(mask), V)
            want = case["packed"]
            ri, gn, cols, vals = a.to_host()
            assert ri.tolist() == want["row_indices"]
            assert gn.tolist() == want["group_ncols"]
            assert cols.tolist() == want["cols"]
            d = sb.decompress(a).cpu().numpy()
            assert np.array_equal(d, W * mask)
        else:
            assert sb.validate_pattern(dev(mask), "shfl_bw", V) == (case["pass"], case["fail_row"])
            if case["status"] == 0:
                sb.compress_shflbw(torch.zeros(m, k, device="cuda"), dev(mask), V)
            else:
                with pytest.raises(sb.NonConformantMask):
                    sb.compress_shflbw(torch.zeros(m, k, device="cuda"), dev(mask), V)


@pytest.mark.parametrize("case", load_golden("full_size.json"),
                         ids=lambda c: f"M{c['M']}K{c['K']}V{c['V']}")
def test_compress_full_size_bit_exact(sb, oracle, case):
    M, K, V = case["M"], case["K"], case["V"]
    mask = oracle.random_shflbw_mask(M, K, V, case["cpg"], oracle.rng(1234))
    W = oracle.round16(oracle.random_dense(M, K, 1))
    a, p = compress_both(sb, oracle, W, mask, V)
    assert digest(p.row_indices) == case["row_indices_digest"]  # oracle pinned to the reference
    assert_same_packing(a, p, oracle)


def test_compress_fp32_dense_rounds_rne(sb, oracle):
    """Unrounded fp32 weights: the converter's bf16 RNE equals the oracle's."""
    mask, _, _ = synthetic(oracle, 256, 512, 8, 32, 0.5)
    W = oracle.random_dense(256, 512, 9)
    a, p = compress_both(sb, oracle, W, mask, 32)
    assert_same_packing(a, p, oracle)


def test_validate_nonconformant_lexicographic(sb, oracle):
    rs = np.random.RandomState(3)
    for t in range(40):
        V = int(rs.randint(2, 5))
        M = V * int(rs.randint(1, 20))
        K = int(rs.randint(1, 150))
        mask = (rs.rand(M, K) < 0.5).astype(np.uint8)
        if t % 3 == 0:  # mostly-conformant: duplicate rows, then break one class
            base = (rs.rand(M // V, K) < 0.3).astype(np.uint8)
            mask = base[rs.permutation(np.repeat(np.arange(M // V), V))]
            mask[rs.randint(M), rs.randint(K)] ^= 1
        assert sb.validate_pattern(dev(mask), "shfl_bw", V) == oracle.validate(mask, V)


def test_mask_entries_must_be_binary(sb):
    mask = torch.ones(4, 4, dtype=torch.uint8, device="cuda")
    mask[1, 2] = 2
    with pytest.raises(sb.BadParams):
        sb.compress_shflbw(torch.zeros(4, 4, device="cuda"), mask, 2)


def test_upload_roundtrip(sb, oracle):
    mask, W, _ = synthetic(oracle, 512, 256, 8, 64, 0.3)
    p = oracle.compress(W, mask, 64)
    a = sb.upload(512, 256, 64, p.row_indices, p.group_ncols, p.cols, p.values)
    assert_same_packing(a, p, oracle)


# ---------------------------------------------------------------- SpMM

def test_spmm_unit_instances_bit_exact(sb, oracle):
    """tests/test_spmm.cpp:115-131 instances (V in {2,4,8}: CUDA-core path),
    bf16 inputs: bit-identical to the reference order."""
    for case in [c for c in load_golden("spmm_random.json") if c["suite"] == "unit"]:
        m, k, n, V = case["m"], case["k"], case["n"], case["V"]
        mask = np.array(case["mask"], np.uint8).reshape(m, k)
        W = oracle.round16(oracle.random_dense(m, k, case["dense_seed"]))
        B = oracle.round16(oracle.random_dense(k, n, case["b_seed"]))
        a, p = compress_both(sb, oracle, W, mask, V)
        got = sb.spmm_execute(a, dev(B, torch.bfloat16)).cpu().numpy()
        assert np.array_equal(got, oracle.spmm(p, B))


def test_spmm_acceptance_instances(sb, oracle):
    """acceptance criterion 1 sequence (tests/acceptance.cpp:59-92): V 2..16."""
    rng = oracle.rng(1001)
    worst = 0.0
    for _ in range(120):
        V = 1 << (1 + rng() % 4)
        m = V * (1 + rng() % (256 // V))
        k = 1 + rng() % 256
        n = 1 + rng() % 64
        alpha = 0.1 * (1 + rng() % 10)
        cpg = int(np.floor(alpha * k + 0.5)) % (k + 1)
        mask = oracle.random_shflbw_mask(m, k, V, cpg, rng)
        W = oracle.round16(oracle.random_dense(m, k, rng()))
        B = oracle.round16(oracle.random_dense(k, n, rng()))
        rng(), rng(), rng()
        a, p = compress_both(sb, oracle, W, mask, V)
        got = sb.spmm_execute(a, dev(B, torch.bfloat16)).cpu().numpy()
        want = oracle.spmm(p, B)
        if V == 16:
            worst = max(worst, oracle.rel_frobenius(got, want))
        else:
            assert np.array_equal(got, want)
    assert worst <= TOL


@pytest.mark.parametrize("M,N,K,V,alpha", [(2048, 128, 2048, 64, 0.25), (2048, 128, 2048, 32, 0.25),
                                           (2048, 128, 2048, 128, 0.25), (4096, 128, 1024, 64, 0.25),
                                           (512, 4096, 2048, 64, 0.25), (2048, 512, 512, 32, 0.5),
                                           (512, 256, 512, 16, 0.5), (2048, 128, 8192, 64, 0.25),
                                           (2048, 256, 4096, 128, 0.1)])
def test_spmm_tc_matches_oracle(sb, oracle, M, N, K, V, alpha):
    mask, W, B = synthetic(oracle, M, K, N, V, alpha)
    a, p = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    n0 = sb.launch_count()
    got = sb.spmm_execute(a, Bd).cpu().numpy()
    assert sb.launch_count() == n0 + 1
    want = oracle.spmm(p, B)
    err = oracle.rel_frobenius(got, want)
    assert err <= TOL, err
    # bf16 output = the same fp32 accumulator rounded once (RNE), bit for bit
    got16 = sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(got16, oracle.round16(got))


def test_spmm_tc_equals_simt_within_tolerance_and_split_is_bitwise(sb, oracle):
    """V-split clusters (multicast) are bit-identical to one CTA per tile;
    K-split clusters (DSMEM reduction in rank order) are deterministic and
    within tolerance."""
    mask, W, B = synthetic(oracle, 2048, 1024, 256, 64, 0.25)
    a, p = compress_both(sb, oracle, W, mask, 64)
    Bd = dev(B, torch.bfloat16)
    want = oracle.spmm(p, B)
    sb.set_option("split", 1)
    base = sb.spmm_execute(a, Bd).cpu().numpy()
    sb.set_option("split_mode", 0)
    for split in (2, 4):
        sb.set_option("split", split)
        assert np.array_equal(sb.spmm_execute(a, Bd).cpu().numpy(), base)
    sb.set_option("split_mode", 1)
    ks = {}
    for split in (2, 4):
        sb.set_option("split", split)
        k1 = sb.spmm_execute(a, Bd).cpu().numpy()
        k2 = sb.spmm_execute(a, Bd).cpu().numpy()
        assert np.array_equal(k1, k2)
        assert oracle.rel_frobenius(k1, want) <= TOL
        ks[split] = k1
    # 2 x 2: the same two K halves as K split by 2, summed in the same order
    sb.set_option("split_mode", 2)
    sb.set_option("split", 4)
    h = sb.spmm_execute(a, Bd).cpu().numpy()
    assert np.array_equal(h, ks[2])
    sb.set_option("split", 0)
    sb.set_option("split_mode", 0)
    sb.set_option("force_simt", 1)
    simt = sb.spmm_execute(a, Bd).cpu().numpy()
    sb.set_option("force_simt", 0)
    assert np.array_equal(simt, want)  # CUDA-core path is bit-exact
    assert oracle.rel_frobenius(base, simt) <= TOL


@pytest.mark.parametrize("split,mode", [(2, 1), (4, 1), (4, 2)])
def test_spmm_ksplit_ragged(sb, oracle, split, mode):
    """K split with groups whose K-block count is not a multiple of the split
    (and empty groups)."""
    rs = np.random.RandomState(21)
    M, K, V, N = 64 * 12, 900, 64, 256
    supports = [np.sort(rs.choice(K, [0, 1, 65, 130, 300, 700][g % 6], replace=False)) for g in range(M // V)]
    perm = rs.permutation(M)
    mask = np.zeros((M, K), np.uint8)
    for r in range(M):
        mask[perm[r], supports[r // V]] = 1
    W = oracle.round16(oracle.random_dense(M, K, 5))
    B = oracle.round16(oracle.random_dense(K, N, 6))
    a, p = compress_both(sb, oracle, W, mask, V)
    sb.set_option("split", split)
    sb.set_option("split_mode", mode)
    got = sb.spmm_execute(a, dev(B, torch.bfloat16)).cpu().numpy()
    sb.set_option("split", 0)
    sb.set_option("split_mode", 0)
    assert oracle.rel_frobenius(got, oracle.spmm(p, B)) <= TOL


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_spmm_ksplit_unaligned_output(sb, oracle, mode, out_dtype):
    """K-split epilogues with per-element stores (output rows not 16-byte
    aligned, so the staged vector-store path is off): same values as the
    aligned path."""
    mask, W, B = synthetic(oracle, 1024, 2048, 136, 64, 0.25)
    a, p = compress_both(sb, oracle, W, mask, 64)
    Bd = dev(B, torch.bfloat16)
    sb.set_option("split", 4)
    sb.set_option("split_mode", mode)
    aligned = sb.spmm_execute(a, Bd, out_dtype=out_dtype)
    big = torch.zeros((1024, 137), dtype=out_dtype, device="cuda")
    sb.spmm_execute(a, Bd, out=big[:, 1:])
    sb.set_option("split", 0)
    sb.set_option("split_mode", 0)
    assert torch.equal(big[:, 1:], aligned)
    assert oracle.rel_frobenius(aligned.float().cpu().numpy(), oracle.spmm(p, B)) <= (TOL if out_dtype == torch.float32 else 1e-2)


@pytest.mark.parametrize("N", [128, 200, 1000])
def test_spmm_cp_async_producers_bitwise(sb, oracle, N):
    """Activation tile filled by TMA gather4, by cp.async (manual 128B
    swizzle), or half/half: identical operands -> identical bits."""
    mask, W, B = synthetic(oracle, 1024, 1024, N, 64, 0.25)
    a, p = compress_both(sb, oracle, W, mask, 64)
    Bd = dev(B, torch.bfloat16)
    sb.set_option("split", 1)
    outs = []
    for cps in (0, 1, 2):
        sb.set_option("cp_async_slabs", cps)
        outs.append(sb.spmm_execute(a, Bd).cpu().numpy())
    sb.set_option("cp_async_slabs", 0)
    sb.set_option("split", 0)
    assert oracle.rel_frobenius(outs[0], oracle.spmm(p, B)) <= TOL
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("N", [8, 136, 200, 1000])
def test_spmm_ragged_n(sb, oracle, N):
    mask, W, B = synthetic(oracle, 1024, 512, N, 64, 0.2)
    a, p = compress_both(sb, oracle, W, mask, 64)
    got = sb.spmm_execute(a, dev(B, torch.bfloat16)).cpu().numpy()
    assert oracle.rel_frobenius(got, oracle.spmm(p, B)) <= TOL


def test_spmm_ragged_and_empty_groups(sb, oracle):
    """groups with different n_g (not multiples of 64) and n_g = 0 (zero rows,
    src/spmm.cpp:103, 115-123)."""
    rs = np.random.RandomState(11)
    M, K, V, N = 64 * 24, 700, 64, 192
    supports = []
    for g in range(M // V):
        n = [0, 1, 63, 64, 65, 130, 700][g % 7]
        supports.append(np.sort(rs.choice(K, n, replace=False)))
    perm = rs.permutation(M)
    mask = np.zeros((M, K), np.uint8)
    for r in range(M):
        mask[perm[r], supports[r // V]] = 1
    W = oracle.round16(oracle.random_dense(M, K, 5))
    B = oracle.round16(oracle.random_dense(K, N, 6))
    a, p = compress_both(sb, oracle, W, mask, V)
    assert_same_packing(a, p, oracle)
    got = sb.spmm_execute(a, dev(B, torch.bfloat16)).cpu().numpy()
    want = oracle.spmm(p, B)
    assert oracle.rel_frobenius(got, want) <= TOL
    zero_rows = [int(r) for g in range(M // V) if p.group_ncols[g] == 0
                 for r in p.row_indices[g * V:(g + 1) * V]]
    assert zero_rows and np.all(got[zero_rows] == 0)


def test_spmm_unaligned_leading_dim_uses_simt(sb, oracle):
    mask, W, B = synthetic(oracle, 256, 128, 13, 64, 0.5)
    a, p = compress_both(sb, oracle, W, mask, 64)
    got = sb.spmm_execute(a, dev(B, torch.bfloat16)).cpu().numpy()
    assert np.array_equal(got, oracle.spmm(p, B))  # N=13: ldb%8 != 0 -> exact path


def test_spmm_fp16(sb, oracle):
    cpg = 128
    mask = oracle.random_shflbw_mask(1024, 512, 64, cpg, oracle.rng(1234))
    W = oracle.round16(oracle.random_dense(1024, 512, 1), "f16")
    B = oracle.round16(oracle.random_dense(512, 256, 2), "f16")
    a = sb.compress_shflbw(dev(W), dev(mask), 64, dtype=torch.float16)
    p = oracle.compress(W, mask, 64)
    got = sb.spmm_execute(a, dev(B, torch.float16)).cpu().numpy()
    assert oracle.rel_frobenius(got, oracle.spmm(p, B)) <= TOL


def test_spmm_shape_errors(sb, oracle):
    mask, W, B = synthetic(oracle, 128, 64, 16, 64, 0.5)
    a, _ = compress_both(sb, oracle, W, mask, 64)
    with pytest.raises(sb.ShapeMismatch):
        sb.spmm_execute(a, torch.zeros(65, 16, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(sb.BadParams):
        sb.spmm_execute(a, dev(B, torch.bfloat16), cfg=sb.TileConfig(t_n=0))
    with pytest.raises(sb.BadParams):
        sb.spmm_execute(a, dev(B, torch.bfloat16), cfg=sb.TileConfig(pipe_stage=1))


def test_sharded_groups_compact_plus_unpermute(sb, oracle):
    """The multi-GPU data path on one device: per-shard compact rows,
    concatenated (what all_gather produces), un-permuted == full SpMM."""
    mask, W, B = synthetic(oracle, 2048, 512, 256, 64, 0.25)
    a, p = compress_both(sb, oracle, W, mask, 64)
    Bd = dev(B, torch.bfloat16)
    full = sb.spmm_execute(a, Bd)
    G = a.group_count()
    for world in (2, 4, 8):
        parts = []
        for rank in range(world):
            g0, g1 = G * rank // world, G * (rank + 1) // world
            out = torch.empty(((g1 - g0) * 64, 256), dtype=torch.float32, device="cuda")
            parts.append(sb.spmm_groups(a, g0, g1, Bd, out, compact=True))
        gathered = torch.cat(parts)
        res = torch.empty_like(full)
        sb.unpermute_rows(a.row_indices_ptr, gathered, res)
        assert torch.equal(res, full)


# ---------------------------------------------------------------- conv

def test_conv_cases_bit_exact(sb, oracle):
    for case in load_golden("conv_cases.json"):
        crs = case["C"] * case["R"] * case["S"]
        mask = np.array(case["mask"], np.uint8).reshape(case["Kf"], crs)
        W = oracle.round16(oracle.random_dense(case["Kf"], crs, case["dense_seed"]))
        x = oracle.round16(oracle.fill_uniform(oracle.rng(case["input_seed"]),
                                               case["C"] * case["H"] * case["W"] * case["Nb"]).reshape(
            case["C"], case["H"], case["W"], case["Nb"]))
        geo = sb.ConvGeometry(case["R"], case["S"], case["stride"], case["pad"])
        a, p = compress_both(sb, oracle, W, mask, case["V"])
        got = sb.conv2d(a, dev(x, torch.bfloat16), geo).cpu().numpy()
        want = oracle.conv2d(p, x, case["R"], case["S"], case["stride"], case["pad"])
        assert np.array_equal(got, want)


@pytest.mark.parametrize("C,H,Kf,R,pad,V,Nb,stride",
                         [(64, 56, 64, 3, 1, 64, 8, 1), (32, 14, 128, 3, 1, 32, 4, 1), (64, 12, 256, 1, 0, 64, 16, 1),
                          (64, 14, 64, 3, 1, 64, 32, 1), (32, 9, 128, 3, 0, 128, 16, 1), (16, 8, 64, 3, 1, 32, 64, 1),
                          (16, 6, 64, 3, 1, 64, 128, 1), (32, 15, 64, 3, 1, 64, 32, 2), (24, 7, 32, 1, 0, 32, 32, 2)])
def test_conv_matches_oracle(sb, oracle, C, H, Kf, R, pad, V, Nb, stride):
    """Implicit-GEMM sparse conv: tcgen05 path when N_b in {16, 32} or a
    multiple of 64, exact CUDA-core path otherwise; padding = TMA zero fill."""
    crs = C * R * R
    mask = oracle.random_shflbw_mask(Kf, crs, V, crs // 4, oracle.rng(1234))
    W = oracle.round16(oracle.random_dense(Kf, crs, 1))
    x = oracle.round16(oracle.fill_uniform(oracle.rng(7), C * H * H * Nb).reshape(C, H, H, Nb))
    a, p = compress_both(sb, oracle, W, mask, V)
    n0 = sb.launch_count()
    got = sb.conv2d(a, dev(x, torch.bfloat16), sb.ConvGeometry(R, R, stride, pad)).cpu().numpy()
    assert sb.launch_count() == n0 + 1
    want = oracle.conv2d(p, x, R, R, stride, pad)
    assert oracle.rel_frobenius(got, want) <= TOL


def test_conv_tc_equals_simt(sb, oracle):
    C, H, Kf, V, Nb = 32, 10, 128, 64, 32
    crs = C * 9
    mask = oracle.random_shflbw_mask(Kf, crs, V, crs // 4, oracle.rng(3))
    W = oracle.round16(oracle.random_dense(Kf, crs, 1))
    x = oracle.round16(oracle.fill_uniform(oracle.rng(5), C * H * H * Nb).reshape(C, H, H, Nb))
    a, p = compress_both(sb, oracle, W, mask, V)
    xd = dev(x, torch.bfloat16)
    tc = sb.conv2d(a, xd, sb.ConvGeometry(3, 3, 1, 1)).cpu().numpy()
    sb.set_option("force_simt", 1)
    simt = sb.conv2d(a, xd, sb.ConvGeometry(3, 3, 1, 1)).cpu().numpy()
    sb.set_option("force_simt", 0)
    assert np.array_equal(simt, oracle.conv2d(p, x, 3, 3, 1, 1))
    assert oracle.rel_frobenius(tc, simt) <= TOL


def test_conv_1x1_equals_spmm_bitwise(sb, oracle):
    C, H, Wd, Nb, Kf, V = 64, 7, 8, 4, 128, 64
    mask = oracle.random_shflbw_mask(Kf, C, V, 16, oracle.rng(3))
    W = oracle.round16(oracle.random_dense(Kf, C, 1))
    x = oracle.round16(oracle.fill_uniform(oracle.rng(4), C * H * Wd * Nb))
    a, _ = compress_both(sb, oracle, W, mask, V)
    xd = dev(x.reshape(C, H, Wd, Nb), torch.bfloat16)
    out = sb.conv2d(a, xd, sb.ConvGeometry())
    ref = sb.spmm_execute(a, xd.reshape(C, H * Wd * Nb))
    assert torch.equal(out.reshape(Kf, -1), ref)


def test_conv_geometry_errors(sb, oracle):
    mask = oracle.random_shflbw_mask(4, 27, 2, 9, oracle.rng(59))
    a = sb.compress_shflbw(dev(oracle.random_dense(4, 27, 1)), dev(mask), 2)
    with pytest.raises(sb.BadGeometry):  # weight cols say C=3, input has C=2
        sb.conv2d(a, torch.zeros(2, 6, 6, 1, device="cuda"), sb.ConvGeometry(3, 3))
    with pytest.raises(sb.BadGeometry):  # (6-3) % 2 != 0
        sb.conv2d(a, torch.zeros(3, 6, 6, 1, device="cuda"), sb.ConvGeometry(3, 3, 2))


@pytest.mark.parametrize("M,N,K,V,alpha,split", [(2048, 4096, 512, 64, 0.25, 0), (512, 2048, 2048, 128, 0.25, 0),
                                                 (1024, 1000, 700, 32, 0.3, 0), (2048, 256, 1024, 64, 0.25, 4),
                                                 (256, 520, 300, 16, 0.5, 0)])
def test_persistent_kernel_bitwise(sb, oracle, M, N, K, V, alpha, split):
    """The persistent kernel (units looped inside a CTA, ping-pong TMEM
    accumulators) computes every unit with the same MMA sequence as the
    one-CTA-per-unit kernel: identical bits, fp32 and bf16 out."""
    mask, W, B = synthetic(oracle, M, K, N, V, alpha)
    a, p = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    sb.set_option("split", split)
    # no K split (its partial sums round differently) and full-width units on
    # the one-CTA-per-unit side, so both kernels run the same MMA sequence
    sb.set_option("split_mode", 3)
    sb.set_option("tile_n", 128)
    outs = {}
    for mode in (-1, 1, 2, 0):  # one CTA per unit, persistent x1 / x2 per SM, auto
        sb.set_option("persistent", mode)
        outs[mode] = (sb.spmm_execute(a, Bd).cpu().numpy(),
                      sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16).float().cpu().numpy())
    sb.set_option("persistent", 2)  # per-element epilogue stores
    sb.set_option("no_bulk_out", 1)
    outs["nb"] = (sb.spmm_execute(a, Bd).cpu().numpy(),
                  sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16).float().cpu().numpy())
    sb.set_option("no_bulk_out", 0)
    sb.set_option("persistent", 0)
    sb.set_option("split", 0)
    sb.set_option("split_mode", 0)
    sb.set_option("tile_n", 0)
    assert oracle.rel_frobenius(outs[1][0], oracle.spmm(p, B)) <= TOL
    for mode in (1, 2, 0, "nb"):
        assert np.array_equal(outs[mode][0], outs[-1][0]) and np.array_equal(outs[mode][1], outs[-1][1]), mode


def test_persistent_conv(sb, oracle):
    C, H, Kf, V, Nb = 32, 12, 128, 64, 32
    crs = C * 9
    mask = oracle.random_shflbw_mask(Kf, crs, V, crs // 4, oracle.rng(8))
    W = oracle.round16(oracle.random_dense(Kf, crs, 1))
    x = oracle.round16(oracle.fill_uniform(oracle.rng(9), C * H * H * Nb).reshape(C, H, H, Nb))
    a, p = compress_both(sb, oracle, W, mask, V)
    xd = dev(x, torch.bfloat16)
    got = {}
    for mode in (1, 2, -1):
        sb.set_option("persistent", mode)
        got[mode] = sb.conv2d(a, xd, sb.ConvGeometry(3, 3, 1, 1)).cpu().numpy()
    sb.set_option("persistent", 0)
    ref = got[-1]
    assert np.array_equal(got[1], ref) and np.array_equal(got[2], ref)
    got = got[1]
    assert oracle.rel_frobenius(got, oracle.conv2d(p, x, 3, 3, 1, 1)) <= TOL


# ------------------------------------------------- permutation folding (§8 f2)

@pytest.mark.parametrize("dtype,V1,V2", [(torch.bfloat16, 64, 32), (torch.float32, 8, 16), (torch.float16, 128, 64)])
def test_fold_input_permutation_chain_bitwise(sb, oracle, dtype, V1, V2):
    """Two chained layers: layer 1 writes group-ordered rows (no write-back
    permutation), layer 2 has row_indices_1 folded into its column indices.
    The final output is bit-identical to the unfolded chain (same gathered
    values, same accumulation order), and on the exact fp32 path equal to the
    oracle chain."""
    M1, K1, M2, N = 1024, 768, 512, 192
    mask1 = oracle.random_shflbw_mask(M1, K1, V1, K1 // 4, oracle.rng(31))
    mask2 = oracle.random_shflbw_mask(M2, M1, V2, M1 // 4, oracle.rng(32))
    W1 = oracle.round16(oracle.random_dense(M1, K1, 33))
    W2 = oracle.round16(oracle.random_dense(M2, M1, 34))
    B = oracle.round16(oracle.random_dense(K1, N, 35))
    a1 = sb.compress_shflbw(dev(W1), dev(mask1), V1, dtype=dtype)
    a2 = sb.compress_shflbw(dev(W2), dev(mask2), V2, dtype=dtype)
    a2f = sb.compress_shflbw(dev(W2), dev(mask2), V2, dtype=dtype)
    Bd = dev(B, dtype)
    odt = torch.float32 if dtype == torch.float32 else dtype
    # unfolded: scatter write-back, then layer 2
    c1 = sb.spmm_execute(a1, Bd, out_dtype=odt)
    want = sb.spmm_execute(a2, c1).cpu().numpy()
    # folded: group-ordered layer-1 rows feed the folded layer 2
    c1p = sb.spmm_execute(a1, Bd, out_dtype=odt, permuted_output=True)
    ri1 = a1.to_host()[0].astype(np.int64)
    assert torch.equal(c1p, c1[torch.from_numpy(ri1).cuda()])
    sb.fold_input_permutation(a2f, a1)
    got = sb.spmm_execute(a2f, c1p).cpu().numpy()
    assert np.array_equal(got, want)
    if dtype == torch.float32:
        p1, p2 = oracle.compress(W1, mask1, V1), oracle.compress(W2, mask2, V2)
        assert np.array_equal(got, oracle.spmm(p2, oracle.spmm(p1, B)))
    # the folded device layout is exactly inv[cols] of the unfolded one
    gp, ci, _ = a2.raw()
    _, cif, _ = a2f.raw()
    inv = np.empty(M1, np.int64)
    inv[ri1] = np.arange(M1)
    assert np.array_equal(cif, np.where(ci >= 0, inv[np.maximum(ci, 0)], -1))


def test_fold_input_permutation_errors(sb, oracle):
    mask = oracle.random_shflbw_mask(128, 256, 32, 64, oracle.rng(3))
    W = oracle.round16(oracle.random_dense(128, 256, 4))
    a = sb.compress_shflbw(dev(W).to(torch.bfloat16), dev(mask), 32)
    before = a.raw()[1].copy()
    bad = torch.arange(256, dtype=torch.int32, device="cuda")
    bad[7] = 3  # duplicate
    with pytest.raises(sb.BadParams):
        sb.fold_input_permutation(a, bad)
    bad[7] = 256  # out of range
    with pytest.raises(sb.BadParams):
        sb.fold_input_permutation(a, bad)
    with pytest.raises(sb.ShapeMismatch):
        sb.fold_input_permutation(a, torch.arange(255, dtype=torch.int32, device="cuda"))
    assert np.array_equal(a.raw()[1], before)  # unchanged on error
    perm = torch.randperm(256, generator=torch.Generator().manual_seed(0)).to(torch.int32).cuda()
    sb.fold_input_permutation(a, perm)
    with pytest.raises(sb.BadParams):  # twice
        sb.fold_input_permutation(a, perm)
    with pytest.raises(sb.BadParams):  # reference-layout download of a folded matrix
        a.to_host()
    x = torch.zeros((16, 4, 4, 32), dtype=torch.bfloat16, device="cuda")  # 16*4*4... C*R*S = 256 = 16*4*4
    with pytest.raises(sb.BadParams):
        sb.conv2d(a, x, sb.ConvGeometry(4, 4, 1, 0))


# ------------------------------------------- conv order (128-byte activation rows)

def _conv_setup(oracle, C, H, Wd, Kf, R, S, V, Nb, seed=5):
    crs = C * R * S
    mask = oracle.random_shflbw_mask(Kf, crs, V, max(1, crs // 4), oracle.rng(seed))
    Wt = oracle.round16(oracle.random_dense(Kf, crs, seed + 1))
    x = oracle.round16(oracle.fill_uniform(oracle.rng(seed + 2), C * H * Wd * Nb).reshape(C, H, Wd, Nb))
    return mask, Wt, x


def test_conv_prepare_layout(sb, oracle):
    """Per group: the same (column, values) pairs, s-runs in ascending s and
    ascending c, every aligned quad of K positions shares one filter column
    s, groups padded to K-tile multiples; decompress is unchanged."""
    C, R, S, Kf, V = 24, 3, 3, 128, 32
    mask, Wt, _ = _conv_setup(oracle, C, 4, 4, Kf, R, S, V, 16)
    w = sb.compress_shflbw(dev(Wt), dev(mask), V)
    wp = sb.conv_prepare(w, sb.ConvGeometry(R, S, 1, 1))
    gp, ci, vv = w.raw()
    gq, cq, vq = wp.raw()
    assert np.all(np.diff(gq) % 64 == 0)
    for g in range(Kf // V):
        a0, a1, b0, b1 = gp[g], gp[g + 1], gq[g], gq[g + 1]
        cols = ci[a0:a1][ci[a0:a1] >= 0]
        got = cq[b0:b1]
        quads = got.reshape(-1, 4)
        for qd in quads:
            v = qd[qd >= 0]
            assert len(set((v % S).tolist())) <= 1
        valid = got[got >= 0]
        want = np.concatenate([np.sort(cols[cols % S == s]) for s in range(S)])
        assert np.array_equal(valid, want)
        src = {int(c): vv[(a0 + j) * V:(a0 + j + 1) * V] for j, c in enumerate(ci[a0:a1]) if c >= 0}
        for j, c in enumerate(got):
            blk = vq[(b0 + j) * V:(b0 + j + 1) * V]
            assert np.array_equal(blk, src[int(c)] if c >= 0 else np.zeros(V, blk.dtype))
    d0 = sb.decompress(w).cpu().numpy()
    d1 = sb.decompress(wp).cpu().numpy()
    assert np.array_equal(d0, d1)
    with pytest.raises(sb.BadParams):
        wp.to_host()


@pytest.mark.parametrize("C,H,Wd,Kf,R,pad,V,Nb", [
    (16, 8, 8, 64, 3, 1, 64, 32),     # 128-byte rows: 2 positions x 32
    (8, 6, 12, 64, 3, 1, 32, 16),     # 4 positions x 16, H != W
    (8, 7, 7, 64, 3, 1, 64, 32),      # Q odd: padded position grid (qp = 8), padding dropped in the epilogue
    (16, 6, 6, 64, 3, 1, 64, 16),     # Nb = 16: 4 positions per row, Q = 6 -> qp = 8
    (8, 9, 5, 64, 3, 1, 64, 32),      # Q = 5, H != W
    (12, 9, 9, 128, 3, 0, 64, 32),    # no padding
    (4, 10, 10, 64, 5, 2, 16, 32),    # 5x5 filter (S = 5)
    (64, 14, 14, 128, 3, 1, 64, 32),  # ResNet-like
])
def test_conv_prepared_matches_oracle(sb, oracle, C, H, Wd, Kf, R, pad, V, Nb):
    mask, Wt, x = _conv_setup(oracle, C, H, Wd, Kf, R, R, V, Nb)
    w = sb.compress_shflbw(dev(Wt), dev(mask), V)
    wp = sb.conv_prepare(w, sb.ConvGeometry(R, R, 1, pad))
    xd = dev(x, torch.bfloat16)
    geo = sb.ConvGeometry(R, R, 1, pad)
    want = oracle.conv2d(oracle.compress(Wt, mask, V), x, R, R, 1, pad)
    got = sb.conv2d(wp, xd, geo).cpu().numpy()
    assert oracle.rel_frobenius(got, want) <= TOL
    base = sb.conv2d(w, xd, geo).cpu().numpy()
    assert oracle.rel_frobenius(got, base) <= TOL
    # persistent kernel: same bits as one CTA per unit
    outs = {}
    for mode in (-1, 2):
        sb.set_option("persistent", mode)
        outs[mode] = sb.conv2d(wp, xd, geo).cpu().numpy()
    sb.set_option("persistent", 0)
    assert np.array_equal(outs[2], outs[-1])
    # CUDA-core path over the conv-ordered layout (pads inside groups)
    sb.set_option("force_simt", 1)
    simt = sb.conv2d(wp, xd, geo).cpu().numpy()
    sb.set_option("force_simt", 0)
    assert oracle.rel_frobenius(simt, want) <= TOL


def test_spmm_with_conv_ordered_matrix(sb, oracle):
    """A conv-ordered matrix is still a valid SpMM operand (pads inside
    groups), on both kernels."""
    mask, Wt, _ = _conv_setup(oracle, 32, 4, 4, 128, 3, 3, 64, 16)
    B = oracle.round16(oracle.random_dense(32 * 9, 256, 77))
    w = sb.compress_shflbw(dev(Wt), dev(mask), 64)
    wp = sb.conv_prepare(w, 3)
    want = oracle.spmm(oracle.compress(Wt, mask, 64), B)
    Bd = dev(B, torch.bfloat16)
    assert oracle.rel_frobenius(sb.spmm_execute(wp, Bd).cpu().numpy(), want) <= TOL
    sb.set_option("force_simt", 1)
    got = sb.spmm_execute(wp, Bd).cpu().numpy()
    sb.set_option("force_simt", 0)
    assert oracle.rel_frobenius(got, want) <= TOL


@pytest.mark.parametrize("prepared", [False, True])
def test_conv_ksplit(sb, oracle, prepared):
    """Conv with its K blocks split over a 2- or 4-CTA cluster (DSMEM
    reduction in K-rank order): deterministic and within tolerance, for both
    activation-row layouts."""
    C, H, Kf, R, pad, V, Nb = 64, 10, 128, 3, 1, 64, 32
    mask, Wt, x = _conv_setup(oracle, C, H, H, Kf, R, R, V, Nb, seed=11)
    w = sb.compress_shflbw(dev(Wt), dev(mask), V)
    if prepared:
        w = sb.conv_prepare(w, R)
    xd = dev(x, torch.bfloat16)
    geo = sb.ConvGeometry(R, R, 1, pad)
    want = oracle.conv2d(oracle.compress(Wt, mask, V), x, R, R, 1, pad)
    for split in (1, 2, 4):
        sb.set_option("split", split)
        a1 = sb.conv2d(w, xd, geo).cpu().numpy()
        a2 = sb.conv2d(w, xd, geo).cpu().numpy()
        assert np.array_equal(a1, a2)
        assert oracle.rel_frobenius(a1, want) <= TOL, split
    sb.set_option("split", 0)


# ---------------------------------------------- SMX1 container <-> device (§8 f1)

@pytest.mark.parametrize("case", [c for c in load_golden("smx1_cases.json") if "M" in c], ids=lambda c: c["name"])
def test_smx1_load_store(sb, oracle, case):
    """Reference-written SMX1 files load straight into the device layout
    (== the oracle's packing of the same matrix), re-encode byte-identically
    with F32 values and to the bf16-rounded file with bf16 values, and
    compute exactly what compress_shflbw's matrix computes."""
    from oracle import smx1_encode
    data = bytes.fromhex(case["hex"])
    mask = oracle.random_shflbw_mask(case["M"], case["K"], case["V"], case["cpg"], oracle.rng(case["mask_seed"]))
    dense = oracle.random_dense(case["M"], case["K"], case["dense_seed"])
    p = oracle.compress(dense, mask, case["V"])
    a32 = sb.smx1_loads(data, torch.float32)
    assert sb.smx1_dumps(a32) == data
    ri, gn, cols, vals = a32.to_host()
    assert np.array_equal(ri, p.row_indices) and np.array_equal(gn, p.group_ncols)
    assert np.array_equal(cols, p.cols) and np.array_equal(vals.view(np.uint32), p.values.view(np.uint32))
    a16 = sb.smx1_loads(data)  # bf16 values
    gp, ci, vv = a16.raw()
    egp, eci, evv = oracle.pack_device(p, 64, "bf16")
    assert np.array_equal(gp, egp) and np.array_equal(ci, eci) and np.array_equal(vv, evv)
    p16 = type(p)(p.M, p.K, p.V, p.row_indices, p.group_ncols, p.cols, oracle.round16(p.values))
    assert sb.smx1_dumps(a16) == smx1_encode(p16)
    # same device matrix as the converter's: identical SpMM bits
    if case["V"] in (16, 32, 64, 128):
        B = oracle.round16(oracle.random_dense(case["K"], 256, 3))
        ac = sb.compress_shflbw(dev(oracle.round16(dense)), dev(mask), case["V"])
        assert np.array_equal(sb.spmm_execute(a16, dev(B, torch.bfloat16)).cpu().numpy(),
                              sb.spmm_execute(ac, dev(B, torch.bfloat16)).cpu().numpy())


def test_smx1_errors_and_files(sb, oracle, tmp_path):
    errs = {7: sb.BadMagic, 8: sb.UnsupportedVersion, 9: sb.CorruptPayload, 3: sb.BadParams}
    for c in load_golden("smx1_cases.json"):
        if c["status"]:
            with pytest.raises(errs[c["status"]]):
                sb.smx1_loads(bytes.fromhex(c["hex"]))
    mask = oracle.random_shflbw_mask(128, 64, 32, 20, oracle.rng(1))
    W = oracle.random_dense(128, 64, 2)
    a = sb.compress_shflbw(dev(W), dev(mask), 32, dtype=torch.float32)
    path = tmp_path / "w.smx1"
    sb.smx1_dump(a, path)
    from oracle import smx1_encode
    assert path.read_bytes() == smx1_encode(oracle.compress(W, mask, 32))
    b = sb.smx1_load(path, torch.float32)
    assert sb.smx1_dumps(b) == path.read_bytes()
    with pytest.raises(sb.BadParams):  # conv-ordered layouts are not the reference's format
        sb.smx1_dumps(sb.conv_prepare(a, 4))


# ------------------------------------------------ pruning on the GPU (§8 f3)

def _prune_scores(oracle, c):
    s = np.abs(oracle.random_dense(c["M"], c["K"], c["score_seed"])).astype(np.float32)
    if c["quantise"]:
        s = (np.floor(s * 4.0) / 4.0).astype(np.float32)
    return s


def _sha(t):
    return hashlib.sha256(np.ascontiguousarray(t.cpu().numpy()).tobytes()).hexdigest()


@pytest.mark.parametrize("case", load_golden("prune_cases.json"), ids=lambda c: c["name"])
def test_prune_shflbw_matches_reference(sb, oracle, case):
    """prune_shflbw and every stage of it equal the reference's results
    (tests/golden/prune_cases.json, written by the compiled reference): masks
    byte for byte, the permutation, and the kept score to the last bit."""
    s = dev(_prune_scores(oracle, case))
    cfg = sb.PruneConfig(**case["cfg"])
    r = sb.prune_shflbw(s, cfg)
    assert _sha(r.mask) == case["mask_digest"]
    assert r.permutation.cpu().tolist() == case["permutation"]
    assert float(r.kept_score).hex() == case["kept_score_hex"]
    um = sb.prune_unstructured(s, cfg.beta())
    assert _sha(um) == case["unstructured_digest"]
    vm = sb.prune_vectorwise(s, cfg.v, cfg.alpha)
    assert _sha(vm) == case["vectorwise_digest"]
    assert float(sb.kept_score(s, vm)).hex() == case["kept_vectorwise_hex"]
    assert sb.kmeans_row_grouping(um, s, cfg).cpu().tolist() == case["kmeans_order"]
    # the pruned mask is a valid Shfl-BW pattern for the converter
    assert sb.validate_pattern(r.mask, "shfl_bw", cfg.v)[0]


def test_prune_fuzz_vs_reference(sb, reference):
    """Random shapes, densities and tie-heavy scores against the compiled
    reference (oracle/_ref travels to the GPU box)."""
    rs = np.random.RandomState(77)
    for t in range(12):
        V = int(rs.choice([1, 2, 4, 8, 16]))
        M = V * int(rs.randint(1, 9))
        K = int(rs.randint(1, 80))
        s = np.abs(rs.randn(M, K)).astype(np.float32)
        if t % 3 == 0:
            s = (np.floor(s * 2) / 2).astype(np.float32)  # many ties, zeros
        cfg = {"alpha": float(rs.choice([0.1, 0.25, 0.5, 0.75, 1.0])), "beta_factor": float(rs.choice([1.0, 2.0, 3.0])),
               "v": V, "kmeans_max_iters": int(rs.choice([1, 5, 50])), "seed": int(rs.randint(0, 100)),
               "restarts": int(rs.randint(1, 4))}
        mask, perm, kept = reference.prune_shflbw(s, cfg)
        r = sb.prune_shflbw(dev(s), sb.PruneConfig(**cfg))
        assert np.array_equal(r.mask.cpu().numpy(), mask), (t, cfg)
        assert np.array_equal(r.permutation.cpu().numpy().astype(np.uint32), perm), (t, cfg)
        assert float(r.kept_score).hex() == float(kept).hex(), (t, cfg)


def test_prune_errors(sb):
    s = torch.ones((8, 8), device="cuda")
    with pytest.raises(sb.BadParams):
        sb.prune_shflbw(s, sb.PruneConfig(alpha=0.0, v=2))
    with pytest.raises(sb.BadParams):
        sb.prune_shflbw(s, sb.PruneConfig(alpha=0.5, v=3))
    with pytest.raises(sb.BadParams):
        sb.prune_shflbw(s, sb.PruneConfig(alpha=0.5, v=2, restarts=0))
    bad = s.clone()
    bad[1, 1] = -1.0
    with pytest.raises(sb.BadParams):
        sb.prune_shflbw(bad, sb.PruneConfig(alpha=0.5, v=2))
    bad[1, 1] = float("nan")
    with pytest.raises(sb.BadParams):
        sb.kept_score(bad, torch.ones((8, 8), dtype=torch.uint8, device="cuda"))
    w = torch.tensor([[-3.0, 2.0]], device="cuda")
    assert sb.importance_scores(w).cpu().tolist() == [[3.0, 2.0]]


@pytest.mark.parametrize("M,N,K,V,alpha,split,mode,persistent",
                         [(2048, 128, 2048, 64, 0.25, 0, 0, 0), (2048, 128, 2048, 64, 0.25, 2, 1, 0),
                          (2048, 128, 2048, 64, 0.25, 4, 3, 0), (1024, 384, 1024, 32, 0.3, 0, 0, -1),
                          (512, 1000, 700, 128, 0.3, 0, 0, -1), (2048, 2048, 512, 64, 0.25, 0, 0, 2),
                          (512, 520, 300, 16, 0.5, 0, 0, 1)])
def test_gather_warps_bitwise(sb, oracle, M, N, K, V, alpha, split, mode, persistent):
    """4 or 8 gather-issuing warps per CTA only change who issues which
    gather4: identical bits in every kernel variant (V/K/2x2 splits,
    persistent), fp32 and bf16 out."""
    mask, W, B = synthetic(oracle, M, K, N, V, alpha)
    a, p = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    sb.set_option("split", split)
    sb.set_option("split_mode", mode)
    sb.set_option("persistent", persistent)
    outs = {}
    for gw in (4, 8):
        sb.set_option("gather_warps", gw)
        outs[gw] = (sb.spmm_execute(a, Bd).cpu().numpy(),
                    sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16).float().cpu().numpy())
    for k, v in (("split", 0), ("split_mode", 0), ("persistent", 0), ("gather_warps", 0)):
        sb.set_option(k, v)
    assert oracle.rel_frobenius(outs[4][0], oracle.spmm(p, B)) <= TOL
    for gw in (8,):
        assert np.array_equal(outs[gw][0], outs[4][0]) and np.array_equal(outs[gw][1], outs[4][1]), gw


@pytest.mark.parametrize("prepared", [False, True])
def test_gather_warps_conv_bitwise(sb, oracle, prepared):
    C, H, Kf, R, pad, V, Nb = 64, 14, 128, 3, 1, 64, 32
    mask, Wt, x = _conv_setup(oracle, C, H, H, Kf, R, R, V, Nb, seed=13)
    w = sb.compress_shflbw(dev(Wt), dev(mask), V)
    if prepared:
        w = sb.conv_prepare(w, R)
    xd = dev(x, torch.bfloat16)
    geo = sb.ConvGeometry(R, R, 1, pad)
    want = oracle.conv2d(oracle.compress(Wt, mask, V), x, R, R, 1, pad)
    outs = {}
    for persistent in (-1, 2):
        sb.set_option("persistent", persistent)
        for gw in (4, 8):
            sb.set_option("gather_warps", gw)
            outs[(persistent, gw)] = sb.conv2d(w, xd, geo).cpu().numpy()
    sb.set_option("persistent", 0)
    sb.set_option("gather_warps", 0)
    ref = outs[(-1, 4)]
    assert oracle.rel_frobenius(ref, want) <= TOL
    for k, v in outs.items():
        assert np.array_equal(v, ref), k


@pytest.mark.parametrize("M,N,K,V,alpha,persistent,split,mode",
                         [(2048, 128, 2048, 64, 0.25, 0, 0, 0),      # 2 x 2 K-split epilogue
                          (512, 4096, 2048, 64, 0.25, -1, 0, 0),     # one CTA per unit, stmatrix staging
                          (2048, 1000, 512, 64, 0.25, 2, 0, 0),      # persistent, ragged last tile
                          (1024, 384, 768, 32, 0.3, 2, 0, 0),        # persistent, V = 32
                          (512, 640, 512, 128, 0.3, -1, 0, 0),       # V = 128 (4 column chunks)
                          (2048, 256, 1024, 64, 0.25, 0, 4, 1)])     # K split by 4
def test_16bit_out_is_rne_of_fp32_out(sb, oracle, M, N, K, V, alpha, persistent, split, mode):
    """Every epilogue (stmatrix-staged tiles, K-split exchange, per-element
    stores) writes bf16 / f16 = the fp32 accumulator rounded once to nearest
    even: bit-identical to rounding the fp32-output result."""
    mask, W, B = synthetic(oracle, M, K, N, V, alpha)
    a, _ = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    sb.set_option("persistent", persistent)
    sb.set_option("split", split)
    sb.set_option("split_mode", mode)
    try:
        c32 = sb.spmm_execute(a, Bd)
        for dt in (torch.bfloat16, torch.float16):
            got = sb.spmm_execute(a, Bd, out_dtype=dt)
            assert torch.equal(got, c32.to(dt)), dt
            sb.set_option("no_bulk_out", 1)
            got_el = sb.spmm_execute(a, Bd, out_dtype=dt)
            sb.set_option("no_bulk_out", 0)
            assert torch.equal(got_el, got), dt
    finally:
        for k in ("persistent", "split", "split_mode", "no_bulk_out"):
            sb.set_option(k, 0)


@pytest.mark.parametrize("M,N,K,V,alpha,persistent,split,mode,world",
                         [(2048, 256, 1024, 64, 0.25, 0, 0, 0, 2),    # auto plan
                          (2048, 128, 2048, 64, 0.25, 0, 4, 2, 2),    # 2 x 2 K-split epilogue
                          (4096, 1024, 512, 64, 0.25, 2, 0, 0, 4),    # persistent
                          (1024, 1000, 768, 32, 0.3, -1, 0, 0, 3),    # ragged N, uneven shards
                          (1024, 512, 512, 128, 0.3, -1, 0, 0, 8)])   # V = 128, 8 destinations
def test_spmm_groups_peers_fused_allgather(sb, oracle, M, N, K, V, alpha, persistent, split, mode, world):
    """The all-gather fused into the epilogue, every destination on this one
    device standing in for a peer GPU: each simulated rank computes its row
    groups once and stores every row into all `world` full-size buffers.
    After all ranks, every buffer equals the single-GPU result bit for bit
    (same kernels, same accumulation order)."""
    mask, W, B = synthetic(oracle, M, K, N, V, alpha)
    a, _ = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    sb.set_option("persistent", persistent)
    sb.set_option("split", split)
    sb.set_option("split_mode", mode)
    try:
        want = sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16)
        full_plan = sb.last_plan()
        outs = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(world)]
        G = a.group_count()
        same = True
        for rank in range(world):
            g0, g1 = G * rank // world, G * (rank + 1) // world
            sb.spmm_groups_peers(a, g0, g1, Bd, outs[rank:] + outs[:rank])  # own buffer first
            # the auto plan of a shard's smaller grid may pick another cluster
            # split than the full grid (a K split sums in another order)
            same &= sb.last_plan().split(" groups=")[0] == full_plan.split(" groups=")[0]
        torch.cuda.synchronize()
        for o in outs:
            if same:
                assert torch.equal(o, want)
            else:  # within one bf16 ulp of the single-GPU result (cancellation
                # results, far below the typical magnitude, within one ulp of rms/64)
                w = want.float()
                mag = torch.maximum(w.abs(), w.pow(2).mean().sqrt() / 64)
                ulp = 2.0 ** (torch.floor(torch.log2(mag)) - 7)
                assert not torch.isnan(o.float()).any()
                assert bool(((o.float() - w).abs() <= ulp).all())
    finally:
        for k in ("persistent", "split", "split_mode"):
            sb.set_option(k, 0)


def test_spmm_groups_peers_errors(sb, oracle):
    mask, W, B = synthetic(oracle, 256, 128, 64, 64, 0.5)
    a, _ = compress_both(sb, oracle, W, mask, 64)
    Bd = dev(B, torch.bfloat16)
    with pytest.raises(sb.BadParams):
        sb.spmm_groups_peers(a, 0, a.group_count(), Bd, [])
    o32 = [torch.zeros((256, 64), dtype=torch.float32, device="cuda")]
    with pytest.raises(sb.Error):  # fp32 output: UNSUPPORTED
        sb.spmm_groups_peers(a, 0, a.group_count(), Bd, o32)
    a32 = sb.compress_shflbw(dev(W), dev(mask), 64, dtype=torch.float32)
    o16 = [torch.zeros((256, 64), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    with pytest.raises(sb.Error):  # exact fp32 matrix: no tcgen05 path, must not silently drop peers
        sb.spmm_groups_peers(a32, 0, a32.group_count(), dev(B), o16)


# ------------------------------------------- unit shape / order variants (round 2)

@pytest.mark.parametrize("N", [128, 72, 200, 1000])
@pytest.mark.parametrize("split,mode", [(1, 0), (2, 1), (4, 1), (2, 3), (4, 2)])
def test_half_width_units_bitwise(sb, oracle, N, split, mode):
    """tile_n = 64 (half-width units: twice the CTAs, each gathering one
    64-column activation slab) computes every output column with the same
    MMA sequence and K-split reduction order as the 128-column units:
    identical bits, fp32 and bf16 out, ragged N included."""
    M, K, V = 1024, 1024, 64
    mask, W, B = synthetic(oracle, M, K, N, V, 0.25)
    a, p = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    sb.set_option("split", split)
    sb.set_option("split_mode", mode)
    outs = {}
    for tn in (128, 64):
        sb.set_option("tile_n", tn)
        outs[tn] = (sb.spmm_execute(a, Bd).cpu().numpy(),
                    sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16).float().cpu().numpy())
        assert f"tile_n={tn}" in sb.last_plan(), sb.last_plan()
    for k in ("tile_n", "split", "split_mode"):
        sb.set_option(k, 0)
    assert np.array_equal(outs[64][0], outs[128][0]) and np.array_equal(outs[64][1], outs[128][1])
    assert oracle.rel_frobenius(outs[64][0], oracle.spmm(p, B)) <= TOL


def test_auto_half_width_north_star_v128(sb, oracle):
    """The auto plan picks half-width units for the V = 128 north-star grid
    (16 groups x 1 column tile: the 128-column plan would use 64 CTAs) and
    stays within tolerance of the oracle."""
    mask, W, B = synthetic(oracle, 2048, 2048, 128, 128, 0.25)
    a, p = compress_both(sb, oracle, W, mask, 128)
    got = sb.spmm_execute(a, dev(B, torch.bfloat16)).cpu().numpy()
    assert "tile_n=64" in sb.last_plan(), sb.last_plan()
    assert oracle.rel_frobenius(got, oracle.spmm(p, B)) <= TOL


@pytest.mark.parametrize("V", [32, 64, 128])
def test_persistent_raster_orders_bitwise(sb, oracle, V):
    """Persistent unit order (group-major vs column-tile-major) changes only
    which CTA computes a unit, never how: identical bits."""
    M, K, N = 4096, 1024, 2048
    mask, W, B = synthetic(oracle, M, K, N, V, 0.25)
    a, p = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    outs = {}
    for r in (1, 2):
        sb.set_option("raster", r)
        outs[r] = sb.spmm_execute(a, Bd).cpu().numpy()
        assert sb.last_plan().startswith("k_spmm_persist") and f"raster={r}" in sb.last_plan(), sb.last_plan()
    sb.set_option("raster", 0)
    assert np.array_equal(outs[1], outs[2])
    assert oracle.rel_frobenius(outs[2][:, :128], oracle.spmm(p, np.ascontiguousarray(B[:, :128]))) <= TOL


@pytest.mark.parametrize("M,K,V,alpha", [(2048, 2048, 64, 0.25),   # 2 x 2 cluster, 4 K blocks per CTA
                                         (4096, 1024, 64, 0.05),   # one K block per CTA
                                         (2048, 2048, 128, 0.25)])  # half-width units
def test_prefetch_and_pdl_trigger_bitwise(sb, oracle, M, K, V, alpha):
    """The L2 prefetch of activation rows before the PDL wait and the PDL
    trigger position change only timing: identical bits for every setting."""
    N = 128
    mask, W, B = synthetic(oracle, M, K, N, V, alpha)
    a, p = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    outs = []
    for pf in (-1, 0, 16):
        for trig in (-1, 1):
            sb.set_option("prefetch", pf)
            sb.set_option("pdl_trigger", trig)
            outs.append(sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16).float().cpu().numpy())
            assert sb.last_plan().startswith("k_spmm_tc"), sb.last_plan()
    sb.set_option("prefetch", 0)
    sb.set_option("pdl_trigger", 0)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    assert oracle.rel_frobenius(outs[0], oracle.spmm(p, B)) <= 1e-2  # bf16 output


@pytest.mark.parametrize("pf,trig", [(16, 1), (16, -1), (-1, 1), (0, 0)])
def test_pdl_chain_consumes_predecessor_output(sb, oracle, pf, trig):
    """Back-to-back SpMMs where each consumes the previous one's output (a
    layer chain: the true data dependency PDL must honour).  With the
    activation prefetch issued before the wait and the trigger at entry, the
    chained results equal the same SpMMs run with a full synchronisation in
    between."""
    M = K = 2048
    N, V = 128, 64
    mats = []
    for i in range(3):
        mask, W, _ = synthetic(oracle, M, K, N, V, 0.25, seed=40 + i)
        mats.append(sb.compress_shflbw(dev(W), dev(mask), V))
    B0 = dev(oracle.round16(np.random.RandomState(9).uniform(-1, 1, (K, N)).astype(np.float32)), torch.bfloat16)
    sb.set_option("prefetch", pf)
    sb.set_option("pdl_trigger", trig)
    try:
        x = B0
        for a in mats:  # enqueued back to back, no host sync
            x = sb.spmm_execute(a, x, out_dtype=torch.bfloat16)
        chained = x.float().cpu().numpy()
        x = B0
        for a in mats:
            x = sb.spmm_execute(a, x, out_dtype=torch.bfloat16)
            torch.cuda.synchronize()
        serial = x.float().cpu().numpy()
    finally:
        sb.set_option("prefetch", 0)
        sb.set_option("pdl_trigger", 0)
    assert np.array_equal(chained, serial)


# ------------------------------------------------- asynchronous converter (round 2)

@pytest.mark.parametrize("M,K,V,alpha", [(2048, 2048, 64, 0.25), (4096, 1024, 32, 0.25), (8192, 1024, 128, 0.1),
                                         (16384, 4096, 64, 0.25), (96, 40, 8, 0.5)])
def test_compress_async_equals_sync(sb, oracle, M, K, V, alpha):
    """shflbw_cu_compress_async (no host sync, bound-sized output) + finalize
    gives the synchronous converter's layout bit for bit, and the SpMM on the
    matrix before finalize is within tolerance of the oracle."""
    cpg = int(np.floor(alpha * K + 0.5))
    mask = oracle.random_shflbw_mask(M, K, V, cpg, oracle.rng(99))
    W = oracle.round16(oracle.random_dense(M, K, 3))
    Wd, md = dev(W), dev(mask)
    a_sync = sb.compress_shflbw(Wd, md, V)
    a, status = sb.compress_shflbw_async(Wd, md, V)
    N = 136
    B = oracle.round16(oracle.random_dense(K, N, 4))
    Bd = dev(B, torch.bfloat16)
    early = sb.spmm_execute(a, Bd).cpu().numpy()  # bound sizes, not finalized yet
    sb.finalize(a, status)
    st = status.cpu().numpy()
    assert st[0] == 0 and st[2] == a_sync.total_cols
    gp, ci, vv = a.raw()
    gq, cq, vq = a_sync.raw()
    assert np.array_equal(gp, gq) and np.array_equal(ci, cq) and np.array_equal(vv, vq)
    ri, gn, cols, vals = a.to_host()
    rj, gm, colsj, valsj = a_sync.to_host()
    assert np.array_equal(ri, rj) and np.array_equal(gn, gm)
    if M * K <= (1 << 24):
        want = oracle.spmm(oracle.compress(W, mask, V), B)
        assert oracle.rel_frobenius(early, want) <= TOL
    assert np.array_equal(sb.spmm_execute(a, Bd).cpu().numpy(), sb.spmm_execute(a_sync, Bd).cpu().numpy())


@pytest.mark.parametrize("M,K,V", [(512, 96, 8), (8192, 128, 32)])  # one-CTA planner, chunked planner
def test_compress_async_reports_errors(sb, oracle, M, K, V):
    """Non-conformant masks and mask bytes > 1 are reported through the
    device status and raised by finalize (the reference's classes and
    fail_row)."""
    mask = oracle.random_shflbw_mask(M, K, V, K // 4, oracle.rng(5))
    mask[7, 3] ^= 1
    want = oracle.validate(mask, V)
    a, status = sb.compress_shflbw_async(torch.zeros(M, K, device="cuda"), dev(mask), V)
    with pytest.raises(sb.NonConformantMask, match=rf"\(row {want[1]}\)"):
        sb.finalize(a, status)
    bad = mask.copy()
    bad[0, 0] = 2
    a, status = sb.compress_shflbw_async(torch.zeros(M, K, device="cuda"), dev(bad), V)
    with pytest.raises(sb.BadParams):
        sb.finalize(a, status)


def test_compress_async_graph_capture(sb, oracle):
    """compress_async + SpMM captured in one CUDA graph: replay after the
    weights change gives the freshly converted product (no host sync inside)."""
    M, K, N, V = 2048, 1024, 256, 64
    mask = oracle.random_shflbw_mask(M, K, V, K // 4, oracle.rng(17))
    md = dev(mask)
    W = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
    B = dev(oracle.round16(oracle.random_dense(K, N, 5)), torch.bfloat16)
    out = torch.empty((M, N), dtype=torch.float32, device="cuda")
    W.copy_(dev(oracle.round16(oracle.random_dense(M, K, 6)), torch.bfloat16))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # the bound-sized matrix + warm-up, outside capture
        a, status = sb.compress_shflbw_async(W, md, V)
        sb.spmm_execute(a, B, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):  # converts into a's buffers on every replay
        sb.compress_shflbw_async(W, md, V, out=a, status=status)
        sb.spmm_execute(a, B, out=out)
    for seed in (7, 8):
        Wn = oracle.round16(oracle.random_dense(M, K, seed))
        W.copy_(dev(Wn, torch.bfloat16))
        g.replay()
        torch.cuda.synchronize()
        want = oracle.spmm(oracle.compress(Wn, mask, V), oracle.round16(oracle.random_dense(K, N, 5)))
        assert oracle.rel_frobenius(out.cpu().numpy(), want) <= TOL
        assert status.cpu().numpy()[0] == 0


# ------------------------------------------- block-wise K blocks: TMA tiles (round 2)

def _bw_mask(M, K, V, keep, seed):
    rs = np.random.RandomState(seed)
    blocks = np.zeros((M // V, K // V), np.uint8)
    for i in range(M // V):
        blocks[i, rs.permutation(K // V)[:keep]] = 1
    return np.kron(blocks, np.ones((V, V), np.uint8))


@pytest.mark.parametrize("M,N,K,keep,persistent", [(1024, 128, 2048, 8, 0), (512, 4096, 2048, 8, 0),
                                                   (2048, 1000, 1024, 4, 2), (1024, 200, 1024, 5, -1)])
def test_blockwise_tile_loads_bitwise(sb, oracle, M, N, K, keep, persistent):
    """Block-wise V x V masks (V = 64): every K block is one contiguous run of
    64 columns, loaded as two TMA 2D tiles instead of 32 gather4s -- the same
    operand bytes in the same layout, so the result is bit-identical to the
    gather path; a mask mixing runs and scattered columns too."""
    V = 64
    mask = _bw_mask(M, K, V, keep, 3)
    if persistent == -1:  # mix: scatter one group's columns
        mask[:V] = 0
        mask[:V, np.random.RandomState(1).choice(K, 96, replace=False)] = 1
    W = oracle.round16(oracle.random_dense(M, K, 1))
    B = oracle.round16(oracle.random_dense(K, N, 2))
    a, p = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    sb.set_option("persistent", persistent if persistent > 0 else 0)
    outs = {}
    for tl in ((0 if persistent != -1 else 1), -1):  # auto (matrix flag) / forced check, gathers only
        sb.set_option("tile_loads", tl)
        outs[tl] = (sb.spmm_execute(a, Bd).cpu().numpy(),
                    sb.spmm_execute(a, Bd, out_dtype=torch.bfloat16).float().cpu().numpy())
    sb.set_option("tile_loads", 0)
    sb.set_option("persistent", 0)
    t = 0 if persistent != -1 else 1
    assert np.array_equal(outs[t][0], outs[-1][0]) and np.array_equal(outs[t][1], outs[-1][1])
    assert oracle.rel_frobenius(outs[t][0][:, :128], oracle.spmm(p, np.ascontiguousarray(B[:, :128]))) <= TOL


def test_persistent_three_per_sm_bitwise(sb, oracle):
    """Many shallow units (FFN1 2048x512, N = 4096): the auto plan runs the
    persistent kernel 3 CTAs per SM (its 64-register instantiation); the
    same units at 2 per SM and on the one-CTA-per-unit kernel give the same
    bits."""
    M, K, N, V = 2048, 512, 4096, 64
    mask, W, B = synthetic(oracle, M, K, N, V, 0.25)
    a, p = compress_both(sb, oracle, W, mask, V)
    Bd = dev(B, torch.bfloat16)
    got3 = sb.spmm_execute(a, Bd).cpu().numpy()
    assert "per_sm=3" in sb.last_plan(), sb.last_plan()
    outs = []
    for opt in (2, -1):
        sb.set_option("persistent", opt)
        outs.append(sb.spmm_execute(a, Bd).cpu().numpy())
    sb.set_option("persistent", 0)
    for o in outs:
        assert np.array_equal(o, got3)
    assert oracle.rel_frobenius(got3[:, :256], oracle.spmm(p, np.ascontiguousarray(B[:, :256]))) <= TOL

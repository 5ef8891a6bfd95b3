"""Pin the C restatement (oracle/shflbw_oracle.c) against the reference.

Every expected value below comes from tests/golden/*.json, which
tests/golden/gen_golden.py produced by running the unmodified reference
(oracle/_ref).  When oracle/_ref is present the last tests also compare the
two libraries directly on fresh random inputs.
"""
import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import OracleError


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits_to_f32(bits):
    return np.array(bits, np.uint32).view(np.float32)


def assert_packed(p, want):
    assert p.row_indices.tolist() == want["row_indices"]
    assert p.group_ncols.tolist() == want["group_ncols"]
    assert p.cols.tolist() == want["cols"]
    assert np.array_equal(p.values.view(np.uint32), np.array(want["values_bits"], np.uint32))


# --- tests/test_formats.cpp known answers --------------------------------

@pytest.mark.parametrize("case", load_golden("formats_kat.json")["compress"], ids=lambda c: c["name"])
def test_compress_known_answers(oracle, case):
    if case["name"] == "shape_mismatch":
        with pytest.raises(OracleError) as e:
            oracle.compress(np.zeros(case["dense_shape"], np.float32),
                            np.zeros(case["mask_shape"], np.uint8), 2)
        assert e.value.code == 1
        return
    dense = bits_to_f32(case["dense_bits"]).reshape(case["dense_shape"])
    mask = np.array(case["mask"], np.uint8).reshape(case["mask_shape"])
    if case["status"] != 0:
        with pytest.raises(OracleError) as e:
            oracle.compress(dense, mask, case["V"])
        assert e.value.code == case["status"]
        if case["status"] == 2:
            assert oracle.validate(mask, case["V"]) == (False, case["fail_row"])
        return
    p = oracle.compress(dense, mask, case["V"])
    assert_packed(p, case["packed"])
    assert np.array_equal(oracle.decompress(p).view(np.uint32).reshape(-1),
                          np.array(case["decompressed_bits"], np.uint32))


def test_known_answers_literal(oracle):
    # tests/test_formats.cpp:14-23, the values spelled out
    p = oracle.compress(np.array([[1, 2], [3, 4]], np.float32), np.ones((2, 2), np.uint8), 2)
    assert p.cols.tolist() == [0, 1] and p.row_indices.tolist() == [0, 1]
    assert p.values.tolist() == [1, 3, 2, 4]


@pytest.mark.parametrize("case", load_golden("formats_kat.json")["stitch"], ids=lambda c: c["name"])
def test_stitch_known_answers(oracle, case):
    from oracle import Packed
    p = Packed(2, case["K"], 2, np.array([0, 1], np.uint32),
               np.array([len(case["cols"])], np.uint32), np.array(case["cols"], np.uint32),
               np.array(case["values"], np.float32))
    tg, tc, tv = oracle.stitch_to_blockwise(p, case["tile_width"])
    assert tg.tolist() == case["tile_group"]
    assert tc.reshape(-1).tolist() == case["tile_cols"]
    assert np.array_equal(tv.reshape(-1).view(np.uint32), np.array(case["tile_values_bits"], np.uint32))


# --- random compress sequences -------------------------------------------

def test_compress_random_sequences(oracle):
    for case in load_golden("compress_random.json"):
        mask = np.array(case["mask"], np.uint8).reshape(case["m"], case["k"])
        if case["suite"] == "roundtrip":
            p = oracle.compress(oracle.random_dense(case["m"], case["k"], case["dense_seed"]), mask,
                                case["V"])
            assert_packed(p, case["packed"])
            assert sorted(p.row_indices.tolist()) == list(range(case["m"]))
        else:
            assert oracle.validate(mask, case["V"]) == (case["pass"], case["fail_row"])
            try:
                oracle.compress(np.zeros((case["m"], case["k"]), np.float32), mask, case["V"])
                st = 0
            except OracleError as e:
                st = e.code
            assert st == case["status"]


def test_generators_match_reference_streams(oracle):
    # the masks stored in the fixtures were drawn by the reference's own
    # test::random_shflbw_mask; redraw the rng-17 spmm sequence
    cases = load_golden("spmm_random.json")
    rng = oracle.rng(17)
    for case in [c for c in cases if c["suite"] == "unit"]:
        v = 1 << (1 + rng() % 3)
        m = v * (1 + rng() % 4)
        k = 1 + rng() % 24
        n = 1 + rng() % 12
        cpg = rng() % (k + 1)
        mask = oracle.random_shflbw_mask(m, k, v, cpg, rng)
        assert (m, k, n, v) == (case["m"], case["k"], case["n"], case["V"])
        assert mask.reshape(-1).tolist() == case["mask"]
        assert rng() == case["dense_seed"]
        assert rng() == case["b_seed"]


# --- SpMM ----------------------------------------------------------------

def test_spmm_unit_instances_bit_exact(oracle):
    for case in [c for c in load_golden("spmm_random.json") if c["suite"] == "unit"]:
        m, k, n, v = case["m"], case["k"], case["n"], case["V"]
        mask = np.array(case["mask"], np.uint8).reshape(m, k)
        a = oracle.compress(oracle.random_dense(m, k, case["dense_seed"]), mask, v)
        B = oracle.random_dense(k, n, case["b_seed"])
        C = oracle.spmm(a, B)
        assert np.array_equal(C.view(np.uint32).reshape(-1), np.array(case["C_bits"], np.uint32))
        # the reference's own tolerance check vs the naive dense oracle
        assert oracle.rel_frobenius(C, oracle.spmm_dense(oracle.decompress(a), B)) <= 1e-5


def test_spmm_acceptance_instances_bit_exact(oracle):
    rng = oracle.rng(1001)
    for case in [c for c in load_golden("spmm_random.json") if c["suite"] == "acceptance1"]:
        v = 1 << (1 + rng() % 4)
        m = v * (1 + rng() % (256 // v))
        k = 1 + rng() % 256
        n = 1 + rng() % 64
        alpha = 0.1 * (1 + rng() % 10)
        cpg = int(np.floor(alpha * k + 0.5)) % (k + 1)
        mask = oracle.random_shflbw_mask(m, k, v, cpg, rng)
        assert digest(mask) == case["mask_digest"]
        assert rng() == case["dense_seed"]
        a = oracle.compress(oracle.random_dense(m, k, case["dense_seed"]), mask, v)
        assert rng() == case["b_seed"]
        B = oracle.random_dense(k, n, case["b_seed"])
        rng(), rng(), rng()  # t_n, t_k, threads
        assert digest(oracle.spmm(a, B)) == case["C_digest"]


def test_spmm_errors(oracle):
    a = oracle.compress(np.eye(2, dtype=np.float32), np.ones((2, 2), np.uint8), 2)
    with pytest.raises(OracleError) as e:
        oracle.spmm(a, np.zeros((3, 2), np.float32))
    assert e.value.code == 1
    # write-back through row_indices, tests/test_spmm.cpp:101-113
    from oracle import Packed
    p = Packed(2, 2, 2, np.array([1, 0], np.uint32), np.array([2], np.uint32),
               np.array([0, 1], np.uint32), np.array([1, 0, 0, 1], np.float32))
    C = oracle.spmm(p, np.array([[5, 6], [7, 8]], np.float32))
    assert C.tolist() == [[7, 8], [5, 6]]


# --- conv ----------------------------------------------------------------

def test_conv_geometry(oracle):
    assert oracle.conv_output_size(6, 6, 3, 3, 1, 0) == (4, 4)
    assert oracle.conv_output_size(6, 6, 3, 3, 1, 1) == (6, 6)
    for args in [(6, 6, 3, 3, 2, 0), (2, 2, 5, 5, 1, 0), (6, 6, 0, 3, 1, 0)]:
        with pytest.raises(OracleError) as e:
            oracle.conv_output_size(*args)
        assert e.value.code == 4


def test_conv_cases(oracle):
    for case in load_golden("conv_cases.json"):
        crs = case["C"] * case["R"] * case["S"]
        mask = np.array(case["mask"], np.uint8).reshape(case["Kf"], crs)
        w = oracle.compress(oracle.random_dense(case["Kf"], crs, case["dense_seed"]), mask, case["V"])
        inp = oracle.fill_uniform(oracle.rng(case["input_seed"]),
                                  case["C"] * case["H"] * case["W"] * case["Nb"]).reshape(
            case["C"], case["H"], case["W"], case["Nb"])
        geo = (case["R"], case["S"], case["stride"], case["pad"])
        out = oracle.conv2d(w, inp, *geo)
        if "out_bits" in case:
            assert np.array_equal(out.view(np.uint32).reshape(-1), np.array(case["out_bits"], np.uint32))
        else:
            assert digest(out) == case["out_digest"]
        direct = oracle.conv_direct(oracle.decompress(w), inp, *geo)
        assert oracle.rel_frobenius(out, direct) <= 1e-5


# --- full-size configurations (digests) -----------------------------------

@pytest.mark.parametrize("case", load_golden("full_size.json"),
                         ids=lambda c: f"M{c['M']}N{c['N']}K{c['K']}V{c['V']}")
def test_full_size_configs(oracle, case):
    M, N, K, V = case["M"], case["N"], case["K"], case["V"]
    mask = oracle.random_shflbw_mask(M, K, V, case["cpg"], oracle.rng(1234))
    assert digest(mask) == case["mask_digest"]
    W = oracle.round16(oracle.random_dense(M, K, 1))
    assert digest(W) == case["W_digest"]
    p = oracle.compress(W, mask, V)
    assert digest(p.row_indices) == case["row_indices_digest"]
    assert digest(p.group_ncols) == case["group_ncols_digest"]
    assert digest(p.cols) == case["cols_digest"]
    assert digest(p.values) == case["values_digest"]
    if "C_digest" in case:
        B = oracle.round16(oracle.random_dense(K, N, 2))
        assert digest(oracle.spmm(p, B)) == case["C_digest"]


# --- direct comparison with the compiled reference ------------------------

def test_oracle_vs_reference_fuzz(oracle, reference):
    """acceptance criterion 7 style fuzz (tests/acceptance.cpp:295-352):
    random masks, validator + compress + spmm agree bit for bit."""
    rs = np.random.RandomState(5)
    for t in range(400):
        v = int(rs.randint(1, 5))
        m = v * int(rs.randint(1, 6))
        k = int(rs.randint(1, 9))
        if t % 2:
            mask = (rs.rand(m, k) < 0.5).astype(np.uint8)
        else:
            g = oracle.rng(t)
            mask = oracle.random_shflbw_mask(m, k, v, int(rs.randint(0, k + 1)), g)
        assert oracle.validate(mask, v) == reference.validate(mask, v)
        dense = oracle.random_dense(m, k, t)
        try:
            p = oracle.compress(dense, mask, v)
        except OracleError as e:
            with pytest.raises(OracleError) as e2:
                reference.compress(dense, mask, v)
            assert e.code == e2.value.code
            continue
        q = reference.compress(dense, mask, v)
        for f in ("row_indices", "group_ncols", "cols", "values"):
            assert np.array_equal(getattr(p, f), getattr(q, f))
        B = oracle.random_dense(k, 1 + t % 7, t + 1)
        assert np.array_equal(oracle.spmm(p, B), reference.spmm(q, B, 1 + t % 5, 1 + t % 3, 1 + t % 3))


def test_rel_frobenius_edge_cases(oracle):
    z = np.zeros(4, np.float32)
    assert oracle.rel_frobenius(z, z) == 0.0
    assert oracle.rel_frobenius(np.ones(4, np.float32), z) == float("inf")


def test_bf16_rounding_rne(oracle):
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e-39], np.float32)
    # 1 + 2^-8 is a tie -> even (1.0); 1 + 3*2^-8 is a tie -> 1 + 2^-6
    y = oracle.round16(x)
    assert y[0] == 1.0 and y[1] == 1.0 and y[2] == np.float32(1.015625) and y[3] == -2.5


# ---------------------------------------------------------------- SMX1 container

def _smx1_source(oracle, c):
    mask = oracle.random_shflbw_mask(c["M"], c["K"], c["V"], c["cpg"], oracle.rng(c["mask_seed"]))
    return oracle.compress(oracle.random_dense(c["M"], c["K"], c["dense_seed"]), mask, c["V"])


def test_smx1_restatement_matches_reference_bytes(oracle):
    """oracle.smx1_encode / smx1_decode (the kind-3 byte format restated)
    against containers written by the reference's encode_container and the
    statuses its decode_container + as_shflbw return."""
    from oracle import smx1_decode, smx1_encode
    for c in load_golden("smx1_cases.json"):
        data = bytes.fromhex(c["hex"])
        st, p = smx1_decode(data)
        assert st == c["status"], c["name"]
        if "M" in c:
            src = _smx1_source(oracle, c)
            assert smx1_encode(src) == data, c["name"]
            assert np.array_equal(p.row_indices, src.row_indices) and np.array_equal(p.cols, src.cols)
            assert np.array_equal(p.values.view(np.uint32), src.values.view(np.uint32))


def test_smx1_restatement_vs_reference_fuzz(oracle, reference):
    """Random valid and single-word-corrupted containers: identical status
    and contents from the restatement and the compiled reference."""
    from oracle import smx1_decode
    rs = np.random.RandomState(5)
    for t in range(60):
        V = int(rs.choice([1, 2, 4, 8]))
        M, K = V * int(rs.randint(1, 6)), int(rs.randint(1, 40))
        mask = reference.random_shflbw_mask(M, K, V, int(rs.randint(0, K + 1)), reference.rng(t))
        data = bytearray(reference.smx1_encode(reference.compress(reference.random_dense(M, K, t), mask, V)))
        if t % 2:
            w = int(rs.randint(0, len(data) // 4))
            data[4 * w:4 * w + 4] = int(rs.randint(0, 2 ** 32)).to_bytes(4, "little")
        data = bytes(data)
        s1, p1 = smx1_decode(data)
        s2, p2 = reference.smx1_decode(data)
        assert s1 == s2, t
        if s1 == 0:
            assert np.array_equal(p1.cols, p2.cols) and np.array_equal(p1.row_indices, p2.row_indices)
            assert np.array_equal(p1.values.view(np.uint32), p2.values.view(np.uint32))


def test_smx1_other_kinds_vs_reference_fuzz(oracle, reference):
    """Containers of the other kinds (dense, mask, vector-wise, block-wise)
    with one random word or length corrupted: the restatement's walk gives the
    reference's status (CorruptPayload, or BadParams for a valid file)."""
    import struct
    from oracle import smx1_decode
    rs = np.random.RandomState(11)

    def hdr(kind, m, k, v, g):
        return b"SMX1" + struct.pack("<6I", 1, kind, m, k, v, g)
    for t in range(400):
        kind = int(rs.choice([0, 1, 2, 4]))
        V = int(rs.choice([1, 2, 4]))
        m, k = V * int(rs.randint(1, 4)), V * int(rs.randint(1, 4))
        if kind == 0:
            body = rs.rand(m * k).astype("<f4").tobytes()
            h = hdr(0, m, k, 0, 0)
        elif kind == 1:
            body = rs.randint(0, 256, (m * k + 7) // 8).astype(np.uint8).tobytes()
            h = hdr(1, m, k, 0, 0)
        elif kind == 2:
            parts = []
            for _ in range(m // V):
                c = np.sort(rs.choice(k, int(rs.randint(0, k + 1)), replace=False)).astype("<u4")
                parts += [struct.pack("<I", len(c)), c.tobytes(), rs.rand(len(c) * V).astype("<f4").tobytes()]
            body = b"".join(parts)
            h = hdr(2, m, k, V, m // V)
        else:
            nbr, nbc = m // V, k // V
            sel = sorted(rs.choice(nbr * nbc, int(rs.randint(0, nbr * nbc + 1)), replace=False))
            body = struct.pack("<I", len(sel)) + b"".join(struct.pack("<II", s // nbc, s % nbc) for s in sel)
            body += rs.rand(len(sel) * V * V).astype("<f4").tobytes()
            h = hdr(4, m, k, V, 0)
        data = bytearray(h + body)
        r = t % 4
        if r == 1 and len(data) > 8:  # one random word
            w = int(rs.randint(2, len(data) // 4))
            data[4 * w:4 * w + 4] = int(rs.choice([0, 1, 2, 3, 7, 2 ** 31, int(rs.randint(0, 2 ** 32))])).to_bytes(4, "little")
        elif r == 2:
            data = data[:int(rs.randint(28, len(data) + 1))]
        elif r == 3:
            data += bytes(int(rs.randint(1, 6)))
        data = bytes(data)
        assert smx1_decode(data)[0] == reference.smx1_decode(data)[0], (t, kind, data.hex())


# ---------------------------------------------------------------- pruning fixtures

def _prune_scores(gen, c):
    s = np.abs(gen.random_dense(c["M"], c["K"], c["score_seed"])).astype(np.float32)
    if c["quantise"]:
        s = (np.floor(s * 4.0) / 4.0).astype(np.float32)
    return s


def test_prune_fixture_scores_regenerate(oracle):
    """The pruning fixtures' importance scores come from the restated
    generator (|random_dense|), so GPU tests rebuild them without the reference."""
    for c in load_golden("prune_cases.json"):
        assert hashlib.sha256(_prune_scores(oracle, c).tobytes()).hexdigest() == c["scores_digest"], c["name"]


def test_prune_fixtures_against_reference(reference):
    for c in load_golden("prune_cases.json"):
        s = _prune_scores(reference, c)
        mask, perm, kept = reference.prune_shflbw(s, c["cfg"])
        assert hashlib.sha256(mask.tobytes()).hexdigest() == c["mask_digest"]
        assert perm.tolist() == c["permutation"] and float(kept).hex() == c["kept_score_hex"]

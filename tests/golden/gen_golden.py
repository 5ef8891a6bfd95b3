"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run (in the build container, where /root/reference exists):

    make -C oracle && python tests/golden/gen_golden.py

Every output value here comes from the unmodified reference library
(oracle/_ref/libshflbw_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  The cases restate the reference's own unit tests
(tests/test_formats.cpp, tests/test_spmm.cpp, tests/test_conv.cpp) and
acceptance criteria 1, 2 and 7 (tests/acceptance.cpp:59-92, 125-186,
295-352), plus the BASELINE.json configurations at full size (as digests).
tests/test_oracle.py then checks the C restatement against these files, and
the GPU parity tests use them as fixtures.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import OracleError, Packed, Reference  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def f32_bits(a: np.ndarray) -> list[int]:
    return np.ascontiguousarray(a, np.float32).view(np.uint32).reshape(-1).tolist()


def packed_json(p: Packed) -> dict:
    return {"row_indices": p.row_indices.tolist(), "group_ncols": p.group_ncols.tolist(),
            "cols": p.cols.tolist(), "values_bits": f32_bits(p.values)}


def status_of(fn):
    try:
        return 0, fn()
    except OracleError as e:
        return e.code, None


def formats_kat(ref: Reference) -> list[dict]:
    """tests/test_formats.cpp:14-135 known-answer cases."""
    cases = []

    def add(name, dense, mask, v):
        dense = np.asarray(dense, np.float32)
        mask = np.asarray(mask, np.uint8)
        st, p = status_of(lambda: ref.compress(dense, mask, v))
        c = {"name": name, "dense_bits": f32_bits(dense), "dense_shape": list(dense.shape),
             "mask": mask.reshape(-1).tolist(), "mask_shape": list(mask.shape), "V": v,
             "status": st}
        if st == 2:
            c["fail_row"] = ref.validate(mask, v)[1]
        if p is not None:
            c["packed"] = packed_json(p)
            c["decompressed_bits"] = f32_bits(ref.decompress(p))
        cases.append(c)

    add("dense_2x2", [[1, 2], [3, 4]], [[1, 1], [1, 1]], 2)
    inter = np.zeros((4, 4), np.uint8)
    inter[[0, 2], 0:2] = 1
    inter[[1, 3], 2:4] = 1
    add("interleaved_4x4", np.arange(1, 17, dtype=np.float32).reshape(4, 4), inter, 2)
    add("diagonal_nonconformant", np.zeros((2, 2)), [[1, 0], [0, 1]], 2)
    add("bad_v", np.zeros((2, 2)), np.zeros((2, 2)), 3)
    add("empty_mask", np.arange(1, 17, dtype=np.float32).reshape(4, 4), np.zeros((4, 4)), 2)
    mult = np.zeros((4, 4), np.uint8)
    mult[[0, 1, 2], 0] = 1
    mult[3, 1] = 1
    add("multiplicity_3_1_v2", np.zeros((4, 4)), mult, 2)
    add("multiplicity_3_1_v1", np.zeros((4, 4)), mult, 1)
    # shape mismatch is checked before anything else (src/formats.cpp:142-143)
    cases.append({"name": "shape_mismatch", "dense_shape": [2, 2], "mask_shape": [2, 3],
                  "status": 1})
    return cases


def stitch_kat(ref: Reference) -> list[dict]:
    """tests/test_formats.cpp:137-181 stitch_to_blockwise cases."""
    out = []
    for name, K, cols, vals, tw in [("sorted", 4, [1, 3], [1, 2, 3, 4], 2),
                                    ("ragged", 8, [0, 4, 7], [1, 1, 2, 2, 3, 3], 2),
                                    ("empty", 4, [], [], 2)]:
        p = Packed(2, K, 2, np.array([0, 1], np.uint32), np.array([len(cols)], np.uint32),
                   np.array(cols, np.uint32), np.array(vals, np.float32))
        tg, tc, tv = ref.stitch_to_blockwise(p, tw)
        out.append({"name": name, "K": K, "cols": cols, "values": vals, "tile_width": tw,
                    "tile_group": tg.tolist(), "tile_cols": tc.reshape(-1).tolist(),
                    "tile_values_bits": f32_bits(tv)})
    return out


def random_compress(ref: Reference) -> list[dict]:
    """Round-trip (tests/test_formats.cpp:183-202, rng 2024) and validation
    soundness (tests/test_formats.cpp:204-225, rng 99) sequences."""
    cases = []
    rng = ref.rng(2024)
    for _ in range(50):
        v = 1 << (rng() % 3)
        m = v * (1 + rng() % 6)
        k = 1 + rng() % 12
        cpg = rng() % (k + 1)
        mask = ref.random_shflbw_mask(m, k, v, cpg, rng)
        dseed = rng()
        dense = ref.random_dense(m, k, dseed)
        p = ref.compress(dense, mask, v)
        cases.append({"suite": "roundtrip", "m": m, "k": k, "V": v, "mask": mask.reshape(-1).tolist(),
                      "dense_seed": dseed, "status": 0, "packed": packed_json(p)})
    rng = ref.rng(99)
    for _ in range(300):
        v = 1 + rng() % 3
        m = v * (1 + rng() % 4)
        k = 1 + rng() % 6
        mask = np.array([rng() % 2 for _ in range(m * k)], np.uint8).reshape(m, k)
        ok, fail_row = ref.validate(mask, v)
        c = {"suite": "soundness", "m": m, "k": k, "V": v, "mask": mask.reshape(-1).tolist(),
             "pass": ok, "fail_row": fail_row}
        st, p = status_of(lambda: ref.compress(np.zeros((m, k), np.float32), mask, v))
        c["status"] = st
        cases.append(c)
    return cases


def spmm_random(ref: Reference) -> list[dict]:
    """tests/test_spmm.cpp:115-131 (rng 17) with full outputs, and acceptance
    criterion 1 (tests/acceptance.cpp:59-92, rng 1001), first 200 instances,
    with output digests."""
    cases = []
    rng = ref.rng(17)
    for _ in range(30):
        v = 1 << (1 + rng() % 3)
        m = v * (1 + rng() % 4)
        k = 1 + rng() % 24
        n = 1 + rng() % 12
        cpg = rng() % (k + 1)
        mask = ref.random_shflbw_mask(m, k, v, cpg, rng)
        dseed = rng()
        a = ref.compress(ref.random_dense(m, k, dseed), mask, v)
        bseed = rng()
        B = ref.random_dense(k, n, bseed)
        Cm = ref.spmm(a, B)
        cases.append({"suite": "unit", "m": m, "k": k, "n": n, "V": v,
                      "mask": mask.reshape(-1).tolist(), "dense_seed": dseed, "b_seed": bseed,
                      "C_bits": f32_bits(Cm)})
    rng = ref.rng(1001)
    for _ in range(200):
        v = 1 << (1 + rng() % 4)
        m = v * (1 + rng() % (256 // v))
        k = 1 + rng() % 256
        n = 1 + rng() % 64
        alpha = 0.1 * (1 + rng() % 10)
        cpg = int(np.floor(alpha * k + 0.5)) % (k + 1)  # llround for positive values
        mask = ref.random_shflbw_mask(m, k, v, cpg, rng)
        dseed = rng()
        a = ref.compress(ref.random_dense(m, k, dseed), mask, v)
        bseed = rng()
        B = ref.random_dense(k, n, bseed)
        t_n = 1 + rng() % 64
        t_k = 1 + rng() % 32
        threads = 1 + rng() % 4
        Cm = ref.spmm(a, B, t_n, t_k, threads)
        cases.append({"suite": "acceptance1", "m": m, "k": k, "n": n, "V": v, "cpg": cpg,
                      "mask_digest": digest(mask), "dense_seed": dseed, "b_seed": bseed,
                      "C_digest": digest(Cm)})
    return cases


def conv_cases(ref: Reference) -> list[dict]:
    """tests/test_conv.cpp:117-139 geometries (rng 47) with full outputs, and
    acceptance criterion 2 (tests/acceptance.cpp:125-186, rng 2002)."""
    cases = []
    rng = ref.rng(47)
    for (c, h, w, n, kf, v, r, s, stride, pad) in [(3, 6, 6, 2, 4, 2, 3, 3, 1, 0),
                                                   (3, 6, 6, 2, 4, 2, 3, 3, 1, 1),
                                                   (2, 7, 7, 1, 4, 4, 3, 3, 2, 0),
                                                   (4, 8, 5, 3, 6, 2, 1, 3, 1, 1),
                                                   (1, 12, 12, 4, 8, 2, 3, 1, 1, 0)]:
        crs = c * r * s
        mask = ref.random_shflbw_mask(kf, crs, v, crs // 2, rng)
        dseed = rng()
        wts = ref.compress(ref.random_dense(kf, crs, dseed), mask, v)
        iseed = rng()
        g = ref.rng(iseed)
        inp = ref.fill_uniform(g, c * h * w * n).reshape(c, h, w, n)
        out = ref.conv2d(wts, inp, r, s, stride, pad)
        cases.append({"suite": "unit", "C": c, "H": h, "W": w, "Nb": n, "Kf": kf, "V": v, "R": r,
                      "S": s, "stride": stride, "pad": pad, "mask": mask.reshape(-1).tolist(),
                      "dense_seed": dseed, "input_seed": iseed, "out_bits": f32_bits(out)})
    rng = ref.rng(2002)
    for i in range(100):
        force = i % 4 == 0
        R = 1 if force else (1 if rng() % 2 else 3)
        S = 1 if force else (1 if rng() % 2 else 3)
        stride = 1 if force else 1 + rng() % 2
        pad = 0 if force else rng() % 2
        while True:
            h = max(R, 1 + rng() % 12)
            w = max(S, 1 + rng() % 12)
            if (h + 2 * pad - R) % stride == 0 and (w + 2 * pad - S) % stride == 0:
                break
        c = 1 + rng() % 8
        v = 1 << (rng() % 3)
        kf = v * (1 + rng() % (8 // v))
        nb = 1 + rng() % 4
        crs = c * R * S
        mask = ref.random_shflbw_mask(kf, crs, v, (crs + 1) // 2, rng)
        dseed = rng()
        wts = ref.compress(ref.random_dense(kf, crs, dseed), mask, v)
        iseed = rng()
        inp = ref.fill_uniform(ref.rng(iseed), c * h * w * nb).reshape(c, h, w, nb)
        rng(), rng()  # cfg.t_n, cfg.t_k draws (results do not depend on them)
        out = ref.conv2d(wts, inp, R, S, stride, pad)
        cases.append({"suite": "acceptance2", "C": c, "H": h, "W": w, "Nb": nb, "Kf": kf, "V": v,
                      "R": R, "S": S, "stride": stride, "pad": pad,
                      "mask": mask.reshape(-1).tolist(), "dense_seed": dseed, "input_seed": iseed,
                      "out_digest": digest(out)})
    return cases


def full_size(ref: Reference) -> list[dict]:
    """BASELINE.json configurations at full size, synthetic inputs per
    SURVEY.md §8(d): mask random_shflbw_mask(M,K,V,llround(alpha*K),
    mt19937_64(1234)), W = random_dense(M,K,1), B = random_dense(K,N,2), both
    rounded to bf16 before the reference sees them.  Digests only."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    orc = Oracle()  # used ONLY for bf16 rounding (a pure bit operation)
    out = []
    for (M, N, K, V, alpha, with_spmm) in [(2048, 128, 2048, 64, 0.25, True),
                                           (2048, 128, 2048, 32, 0.25, True),
                                           (2048, 128, 2048, 128, 0.25, True),
                                           (4096, 128, 1024, 64, 0.25, True),
                                           (512, 256, 512, 64, 0.5, True),
                                           (2048, 64, 512, 32, 0.1, True),
                                           # large FFN (M > 4096: the converter's multi-block radix sort)
                                           (16384, 8192, 4096, 64, 0.25, False),
                                           (8192, 128, 2048, 32, 0.25, False),
                                           (8192, 128, 1024, 128, 0.1, False)]:
        cpg = int(np.floor(alpha * K + 0.5))
        mask = ref.random_shflbw_mask(M, K, V, cpg, ref.rng(1234))
        W = orc.round16(ref.random_dense(M, K, 1))
        p = ref.compress(W, mask, V)
        case = {"M": M, "N": N, "K": K, "V": V, "alpha": alpha, "cpg": cpg,
                "mask_digest": digest(mask), "W_digest": digest(W),
                "row_indices_digest": digest(p.row_indices), "group_ncols_digest": digest(p.group_ncols),
                "cols_digest": digest(p.cols), "values_digest": digest(p.values)}
        if with_spmm:
            B = orc.round16(ref.random_dense(K, N, 2))
            case["C_digest"] = digest(ref.spmm(p, B, threads=8))
        out.append(case)
    return out


def smx1_cases(ref: Reference) -> list[dict]:
    """SMX1 kind-3 containers written by the reference's encode_container
    (src/container.cpp:141-145) and the statuses its decode_container +
    as_shflbw give for valid and corrupted files (src/container.cpp:147-215)."""
    out = []
    for name, m, k, v, cpg, mseed, dseed in [("small", 64, 96, 8, 24, 3, 4), ("v1", 12, 10, 1, 3, 5, 6),
                                           ("empty_groups", 32, 40, 16, 0, 7, 8), ("v64", 128, 96, 64, 20, 9, 10),
                                           ("tiny", 16, 12, 4, 3, 12, 13)]:
        mask = ref.random_shflbw_mask(m, k, v, cpg, ref.rng(mseed))
        p = ref.compress(ref.random_dense(m, k, dseed), mask, v)
        b = ref.smx1_encode(p)
        out.append({"name": name, "M": m, "K": k, "V": v, "cpg": cpg, "mask_seed": mseed, "dense_seed": dseed,
                    "hex": b.hex(), "status": ref.smx1_decode(b)[0]})
    base = bytes.fromhex(out[-1]["hex"])  # the tiny matrix
    M, V, K = 16, 4, 12
    ri_off = 28
    g0 = ri_off + 4 * M  # first group record
    def patch(b, off, val):
        return b[:off] + int(val).to_bytes(4, "little") + b[off + 4:]
    bad = {
        "bad_magic": b"SMX2" + base[4:],
        "short_magic": base[:3],
        "version_2": patch(base, 4, 2),
        "truncated_header": base[:20],
        "truncated_payload": base[:-3],
        "trailing_byte": base + b"\0",
        "unknown_kind": patch(base, 8, 7),
        "dense_kind": ref.smx1_encode_dense(ref.random_dense(3, 5, 11)),
        "row_indices_duplicate": patch(base, ri_off + 4, int.from_bytes(base[ri_off:ri_off + 4], "little")),
        "row_index_out_of_range": patch(base, ri_off, M),
        "vg_mismatch": patch(base, 24, M // V + 1),
        "v_zero": patch(base, 20, 0),
        "ncols_exceeds_k": patch(base, g0, K + 1),
        "col_out_of_range": patch(base, g0 + 4, K),
        "cols_not_increasing": patch(base, g0 + 8, int.from_bytes(base[g0 + 4:g0 + 8], "little")),
    }
    # other kinds: the reference decodes (and validates) the payload before
    # as_shflbw rejects the kind, so a corrupt one is CorruptPayload
    import struct

    def hdr(kind, m, k, v, g):
        return b"SMX1" + struct.pack("<6I", 1, kind, m, k, v, g)

    def f32(*xs):
        return struct.pack(f"<{len(xs)}f", *xs)

    def u32(*xs):
        return struct.pack(f"<{len(xs)}I", *xs)
    dense_ok = ref.smx1_encode_dense(ref.random_dense(2, 3, 11))
    vw_ok = hdr(2, 4, 5, 2, 2) + u32(2, 0, 3) + f32(1, 2, 3, 4) + u32(1, 4) + f32(5, 6)
    bw_ok = hdr(4, 4, 4, 2, 0) + u32(2, 0, 1, 1, 0) + f32(*range(8))
    bad.update({
        "dense_truncated": dense_ok[:-4],
        "dense_trailing": dense_ok + b"\0\0\0\0",
        "dense_nan": dense_ok[:-4] + f32(float("nan")),
        "dense_inf": dense_ok[:32] + f32(float("inf")) + dense_ok[36:],
        "mask_ok": hdr(1, 3, 5, 0, 0) + bytes([0b01001001, 0b0101]),
        "mask_truncated": hdr(1, 3, 5, 0, 0) + bytes([0b01001001]),
        "mask_trailing": hdr(1, 3, 5, 0, 0) + bytes([1, 2, 3]),
        "vw_ok": vw_ok,
        "vw_vg_mismatch": hdr(2, 4, 5, 2, 3) + vw_ok[28:],
        "vw_v_zero": hdr(2, 4, 5, 0, 2) + vw_ok[28:],
        "vw_cols_not_increasing": hdr(2, 4, 5, 2, 2) + u32(2, 3, 3) + f32(1, 2, 3, 4) + u32(1, 4) + f32(5, 6),
        "vw_col_out_of_range": hdr(2, 4, 5, 2, 2) + u32(2, 0, 5) + f32(1, 2, 3, 4) + u32(1, 4) + f32(5, 6),
        "vw_ncols_exceeds_k": hdr(2, 4, 5, 2, 2) + u32(6) + vw_ok[32:],
        "vw_truncated": vw_ok[:-2],
        "vw_trailing": vw_ok + b"\0",
        "bw_ok": bw_ok,
        "bw_v_not_dividing": hdr(4, 4, 5, 2, 0) + bw_ok[28:],
        "bw_v_zero": hdr(4, 4, 4, 0, 0) + bw_ok[28:],
        "bw_coord_out_of_range": hdr(4, 4, 4, 2, 0) + u32(2, 0, 1, 2, 0) + f32(*range(8)),
        "bw_coords_unsorted": hdr(4, 4, 4, 2, 0) + u32(2, 1, 0, 0, 1) + f32(*range(8)),
        "bw_coords_duplicate": hdr(4, 4, 4, 2, 0) + u32(2, 0, 1, 0, 1) + f32(*range(8)),
        "bw_truncated_coords": hdr(4, 4, 4, 2, 0) + u32(2, 0, 1, 1),
        "bw_truncated_values": bw_ok[:-4],
        "bw_trailing": bw_ok + b"\0",
        "bw_missing_count": hdr(4, 4, 4, 2, 0),
    })
    for name, b in bad.items():
        out.append({"name": name, "hex": b.hex(), "status": ref.smx1_decode(b)[0]})
    return out


PRUNE_CASES = [  # name, M, K, V, alpha, beta_factor, iters, seed, restarts, score seed, quantise
    ("small", 8, 12, 2, 0.5, 2.0, 50, 0, 4, 1, False),
    ("ties", 16, 16, 4, 0.25, 2.0, 50, 3, 4, 2, True),
    ("v1_topk", 6, 10, 1, 0.3, 2.0, 50, 0, 2, 3, False),
    ("single_group", 8, 20, 8, 0.25, 2.0, 50, 1, 2, 4, False),
    ("alpha_one", 8, 8, 4, 1.0, 2.0, 50, 0, 2, 5, False),
    ("mid", 64, 96, 8, 0.25, 2.0, 50, 7, 4, 6, False),
    ("mid_ties", 60, 40, 6, 0.3, 1.5, 20, 11, 3, 7, True),
    ("wide", 128, 256, 16, 0.25, 2.0, 50, 2, 4, 8, False),
    ("v64", 256, 512, 64, 0.25, 2.0, 50, 5, 2, 9, False),
]


def prune_scores(ref_or_orc, M, K, sseed, quantise):
    """importance scores for the pruning fixtures: |random_dense| (the
    reference's generator), optionally quantised to quarters so that ties
    exercise every tie-break rule."""
    s = np.abs(ref_or_orc.random_dense(M, K, sseed)).astype(np.float32)
    if quantise:
        s = (np.floor(s * 4.0) / 4.0).astype(np.float32)
    return s


def prune_cases(ref: Reference) -> list[dict]:
    """prune_shflbw and its parts (src/pruning.cpp) on the reference."""
    out = []
    for (name, M, K, V, alpha, bf, iters, seed, restarts, sseed, quant) in PRUNE_CASES:
        s = prune_scores(ref, M, K, sseed, quant)
        cfg = {"alpha": alpha, "beta_factor": bf, "v": V, "kmeans_max_iters": iters, "seed": seed,
               "restarts": restarts}
        mask, perm, kept = ref.prune_shflbw(s, cfg)
        beta = min(1.0, bf * alpha)
        um = ref.prune_unstructured(s, beta)
        vm = ref.prune_vectorwise(s, V, alpha)
        order = ref.kmeans_row_grouping(um, s, cfg)
        out.append({"name": name, "M": M, "K": K, "cfg": cfg, "score_seed": sseed, "quantise": quant,
                    "scores_digest": digest(s),
                    "mask_digest": digest(mask), "mask_popcount": int(mask.sum()),
                    "permutation": perm.tolist(), "kept_score_hex": float(kept).hex(),
                    "unstructured_digest": digest(um), "vectorwise_digest": digest(vm),
                    "kmeans_order": order.tolist(),
                    "kept_vectorwise_hex": float(ref.kept_score(s, vm)).hex()})
    return out


def main() -> None:
    ref = Reference()
    files = {
        "formats_kat.json": {"compress": formats_kat(ref), "stitch": stitch_kat(ref)},
        "compress_random.json": random_compress(ref),
        "spmm_random.json": spmm_random(ref),
        "conv_cases.json": conv_cases(ref),
        "full_size.json": full_size(ref),
        "smx1_cases.json": smx1_cases(ref),
        "prune_cases.json": prune_cases(ref),
    }
    only = sys.argv[1:]
    files = {k: v for k, v in files.items() if not only or k in only}
    for name, obj in files.items():
        with open(os.path.join(HERE, name), "w") as f:
            json.dump({"generator": "tests/golden/gen_golden.py (reference: oracle/_ref)",
                       "cases": obj}, f, separators=(",", ":"))
        print(name, os.path.getsize(os.path.join(HERE, name)), "bytes")


if __name__ == "__main__":
    main()

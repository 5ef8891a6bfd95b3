// container.cpp -- SMX1 kind-3 (Shfl-BW) container <-> device packed layout
// (SURVEY.md §8 f1).  The byte format is the reference's
// (include/shflbw/container.hpp:14-22): "SMX1", u32 version 1, kind, M, K, V,
// G, then M u32 row_indices and per group u32 n_g, n_g u32 columns, V*n_g
// f32 values, little-endian.
//
//   shflbw_cu_smx1_decode  replaces decode_container + as_shflbw
//                          (src/container.cpp:147-215, :90-124, :126-134)
//                          followed by an upload: the payload is validated
//                          with the reference's rules and error classes, the
//                          group records are de-interleaved once on the host
//                          and uploaded straight into the padded device
//                          layout (values rounded to the requested dtype).
//   shflbw_cu_smx1_encode  replaces encode_container(ShflBWMatrix)
//                          (src/container.cpp:141-145, :82-88) for a device
//                          matrix: byte-identical to the reference's file for
//                          the same (exact) values.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "shflbw_cu.h"

namespace sbw {
int fail(int code, const std::string& msg);  // capi.cu
}

namespace {

constexpr char kMagic[4] = {'S', 'M', 'X', '1'};
constexpr uint32_t kKindShflBW = 3;

struct Reader {
    const uint8_t* p;
    uint64_t n, pos = 0;
    bool ok = true;
    uint32_t u32() {
        if (n - pos < 4) {
            ok = false;
            return 0;
        }
        uint32_t v;
        std::memcpy(&v, p + pos, 4);  // little-endian host (x86-64 / aarch64)
        pos += 4;
        return v;
    }
    // n 32-bit words into dst (bounds-checked before copying)
    bool words(void* dst, uint64_t count) {
        if (count > (n - pos) / 4) {
            ok = false;
            return false;
        }
        if (count) std::memcpy(dst, p + pos, count * 4);
        pos += count * 4;
        return true;
    }
};

void put(std::vector<uint8_t>& out, const void* src, size_t bytes) {
    const auto* b = static_cast<const uint8_t*>(src);
    out.insert(out.end(), b, b + bytes);
}

// Walks the payload of another valid kind (0 dense, 1 mask, 2 vector-wise,
// 4 block-wise) with the reference's checks, in the reference's order
// (decode_container, src/container.cpp:158-238): nothing is materialised.
// Returns the CorruptPayload message, or nullptr if the file decodes (the
// caller then fails as_shflbw's kind check with BadParams, src/container.cpp:126-134).
const char* walk_other_kind(Reader& r, uint32_t kind, uint32_t m, uint32_t k, uint32_t v, uint32_t g) {
    static const char* kTrunc = "container truncated";
    auto done = [&]() -> const char* { return r.pos != r.n ? "trailing bytes after payload" : nullptr; };
    auto skip_f32s = [&](uint64_t count) -> bool {  // Reader::f32s: count > remaining / 4 -> truncated
        if (count > (r.n - r.pos) / 4) return false;
        r.pos += count * 4;
        return true;
    };
    switch (kind) {
        case 0: {  // dense: values, then trailing bytes, then finiteness
            const uint64_t count = static_cast<uint64_t>(m) * k;
            const uint64_t start = r.pos;
            if (!skip_f32s(count)) return kTrunc;
            if (const char* e = done()) return e;
            for (uint64_t i = 0; i < count; ++i) {
                uint32_t bits;
                std::memcpy(&bits, r.p + start + 4 * i, 4);
                if ((bits & 0x7f800000u) == 0x7f800000u) return "dense payload holds non-finite value";
            }
            return nullptr;
        }
        case 1: {  // mask: ceil(m*k / 8) packed bytes
            const uint64_t nbytes = (static_cast<uint64_t>(m) * k + 7) / 8;
            if (r.pos + nbytes > r.n) return kTrunc;
            r.pos += nbytes;
            return done();
        }
        case 2: {  // vector-wise: read_vector_wise_payload (src/container.cpp:90-115)
            if (v == 0 || static_cast<uint64_t>(v) * g != m) return "vector-wise header: V * G != M";
            for (uint32_t gi = 0; gi < g; ++gi) {
                const uint32_t ng = r.u32();
                if (!r.ok) return kTrunc;
                if (ng > k) return "group column count exceeds K";
                uint32_t prev = 0;
                for (uint32_t j = 0; j < ng; ++j) {
                    const uint32_t c = r.u32();
                    if (!r.ok) return kTrunc;
                    if (c >= k || (j > 0 && c <= prev)) return "group columns must be strictly increasing and < K";
                    prev = c;
                }
                if (!skip_f32s(static_cast<uint64_t>(ng) * v)) return kTrunc;
            }
            return done();
        }
        case 4: {  // block-wise (src/container.cpp:213-235)
            if (v == 0 || m % v != 0 || k % v != 0) return "block-wise header: V must divide M and K";
            const uint32_t nblocks = r.u32();
            if (!r.ok) return kTrunc;
            if (r.pos + static_cast<uint64_t>(nblocks) * 8 > r.n) return kTrunc;
            uint32_t pbr = 0, pbc = 0;
            for (uint32_t b = 0; b < nblocks; ++b) {
                const uint32_t br = r.u32(), bc = r.u32();
                if (br >= m / v || bc >= k / v) return "block coordinate out of range";
                if (b > 0 && (br < pbr || (br == pbr && bc <= pbc))) return "block coordinates must be sorted and unique";
                pbr = br;
                pbc = bc;
            }
            // size_t(nblocks) * v * v, with the reference's 64-bit wrap-around
            if (!skip_f32s(static_cast<uint64_t>(nblocks) * v * v)) return kTrunc;
            return done();
        }
    }
    return "unknown container kind";
}

}  // namespace

extern "C" {

int shflbw_cu_smx1_decode(const void* bytes, uint64_t nbytes, int32_t value_dtype, shflbw_cu_matrix* out,
                          shflbw_stream_t stream) {
    using sbw::fail;
    if (!out || (!bytes && nbytes)) return fail(SHFLBW_BAD_PARAMS, "smx1_decode: null argument");
    const auto* b = static_cast<const uint8_t*>(bytes);
    if (nbytes < 4 || std::memcmp(b, kMagic, 4) != 0) return fail(SHFLBW_BAD_MAGIC, "not an SMX1 container");
    Reader r{b, nbytes, 4};
    const uint32_t version = r.u32();
    if (!r.ok) return fail(SHFLBW_CORRUPT_PAYLOAD, "container truncated");
    if (version != 1) return fail(SHFLBW_UNSUPPORTED_VERSION, "SMX1 version " + std::to_string(version));
    const uint32_t kind = r.u32(), M = r.u32(), K = r.u32(), V = r.u32(), G = r.u32();
    if (!r.ok) return fail(SHFLBW_CORRUPT_PAYLOAD, "container truncated");
    if (kind <= 4 && kind != kKindShflBW) {
        // another kind: decoded (and validated) first, as the reference's
        // decode_container does; a valid one then fails as_shflbw (BadParams)
        if (const char* e = walk_other_kind(r, kind, M, K, V, G)) return fail(SHFLBW_CORRUPT_PAYLOAD, e);
        return fail(SHFLBW_BAD_PARAMS, "container holds kind " + std::to_string(kind) + ", not a Shfl-BW matrix");
    }
    if (kind != kKindShflBW) return fail(SHFLBW_CORRUPT_PAYLOAD, "unknown container kind " + std::to_string(kind));
    // sizes are checked against the bytes present before anything is allocated
    if (static_cast<uint64_t>(M) > (nbytes - r.pos) / 4) return fail(SHFLBW_CORRUPT_PAYLOAD, "container truncated");
    std::vector<uint32_t> row_indices(M);
    if (!r.words(row_indices.data(), M)) return fail(SHFLBW_CORRUPT_PAYLOAD, "container truncated");
    {
        std::vector<uint8_t> seen(M, 0);
        for (uint32_t x : row_indices) {
            if (x >= M || seen[x]) return fail(SHFLBW_CORRUPT_PAYLOAD, "row_indices is not a permutation of 0..M-1");
            seen[x] = 1;
        }
    }
    if (V == 0 || static_cast<uint64_t>(V) * G != M) return fail(SHFLBW_CORRUPT_PAYLOAD, "vector-wise header: V * G != M");
    if (M > 0x7fffffffu || K > 0x7fffffffu) return fail(SHFLBW_UNSUPPORTED, "smx1_decode: M or K exceeds 2^31");
    std::vector<uint32_t> group_ncols(G), cols;
    std::vector<float> values;
    for (uint32_t g = 0; g < G; ++g) {
        const uint32_t ng = r.u32();
        if (!r.ok) return fail(SHFLBW_CORRUPT_PAYLOAD, "container truncated");
        if (ng > K) return fail(SHFLBW_CORRUPT_PAYLOAD, "group column count exceeds K");
        group_ncols[g] = ng;
        if ((static_cast<uint64_t>(ng) * (1 + V)) > (nbytes - r.pos) / 4)
            return fail(SHFLBW_CORRUPT_PAYLOAD, "container truncated");
        const size_t c0 = cols.size();
        cols.resize(c0 + ng);
        if (!r.words(cols.data() + c0, ng)) return fail(SHFLBW_CORRUPT_PAYLOAD, "container truncated");
        for (uint32_t j = 0; j < ng; ++j)
            if (cols[c0 + j] >= K || (j > 0 && cols[c0 + j] <= cols[c0 + j - 1]))
                return fail(SHFLBW_CORRUPT_PAYLOAD, "group columns must be strictly increasing and < K");
        const size_t v0 = values.size();
        values.resize(v0 + static_cast<size_t>(ng) * V);
        if (!r.words(values.data() + v0, static_cast<uint64_t>(ng) * V))
            return fail(SHFLBW_CORRUPT_PAYLOAD, "container truncated");
    }
    if (r.pos != nbytes) return fail(SHFLBW_CORRUPT_PAYLOAD, "trailing bytes after payload");
    return shflbw_cu_matrix_upload(static_cast<int32_t>(M), static_cast<int32_t>(K), static_cast<int32_t>(V),
                                   row_indices.data(), group_ncols.data(), cols.data(), values.data(), value_dtype,
                                   out, stream);
}

int shflbw_cu_smx1_encode(const shflbw_cu_matrix* m, void* bytes, uint64_t capacity, uint64_t* nbytes,
                          shflbw_stream_t stream) {
    using sbw::fail;
    if (!m || !nbytes) return fail(SHFLBW_BAD_PARAMS, "smx1_encode: null argument");
    if (m->rows < 0 || m->v <= 0 || m->groups < 0) return fail(SHFLBW_BAD_PARAMS, "smx1_encode: invalid matrix");
    const uint32_t M = static_cast<uint32_t>(m->rows), G = static_cast<uint32_t>(m->groups), V = m->v;
    std::vector<uint32_t> row_indices(M ? M : 1), group_ncols(G ? G : 1);
    // sizes first: the column total is the sum of n_g
    const uint64_t cap_cols = m->total_cols > 0 ? static_cast<uint64_t>(m->total_cols) : 1;
    std::vector<uint32_t> cols(cap_cols);
    std::vector<float> values(cap_cols * V);
    if (int st = shflbw_cu_matrix_download(m, row_indices.data(), group_ncols.data(), cols.data(), values.data(),
                                           stream))
        return st;
    uint64_t total = 0;
    for (uint32_t g = 0; g < G; ++g) total += group_ncols[g];
    const uint64_t size = 28 + 4ull * M + 4ull * G + 4ull * total + 4ull * total * V;
    *nbytes = size;
    if (!bytes) return SHFLBW_OK;  // size query
    if (capacity < size) return fail(SHFLBW_BAD_PARAMS, "smx1_encode: buffer too small");
    std::vector<uint8_t> out;
    out.reserve(size);
    put(out, kMagic, 4);
    const uint32_t hdr[6] = {1, kKindShflBW, M, static_cast<uint32_t>(m->cols), V, G};
    put(out, hdr, sizeof(hdr));
    put(out, row_indices.data(), 4ull * M);
    uint64_t off = 0;
    for (uint32_t g = 0; g < G; ++g) {
        const uint32_t ng = group_ncols[g];
        put(out, &ng, 4);
        put(out, cols.data() + off, 4ull * ng);
        put(out, values.data() + off * V, 4ull * ng * V);
        off += ng;
    }
    std::memcpy(bytes, out.data(), out.size());
    return SHFLBW_OK;
}

}  // extern "C"

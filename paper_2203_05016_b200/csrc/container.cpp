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
    if (kind <= 4 && kind != kKindShflBW)  // a valid other kind: the reference's as_shflbw throws BadParams
        return fail(SHFLBW_BAD_PARAMS, "container holds kind " + std::to_string(kind) + ", not a Shfl-BW matrix");
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

// ref_shim.cpp -- extern "C" face of the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together
// with the reference's own sources where they lie
// (/root/reference/proj/src/{matrix,formats,spmm,rng,container,pruning}.cpp) into
// oracle/_ref/libshflbw_ref.so.  It is used (a) to generate and re-check the
// golden fixtures under tests/golden/, (b) to pin the C restatement in
// oracle/shflbw_oracle.c, and (c) as bench.py's `--impl reference` arm (the
// reference's own CPU spmm_execute / conv2d, all host threads).
//
// Flat array conventions follow oracle/shflbw_oracle.h.  Return codes (the
// library's, include/shflbw_cu.h): 0 ok, 1 ShapeMismatch, 2 NonConformantMask,
// 3 BadParams, 4 BadGeometry, 7 BadMagic, 8 UnsupportedVersion,
// 9 CorruptPayload, 99 other shflbw::Error.
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "shflbw/container.hpp"
#include "shflbw/formats.hpp"
#include "shflbw/pruning.hpp"
#include "shflbw/rng.hpp"
#include "shflbw/spmm.hpp"
#include "test_helpers.hpp"

using namespace shflbw;

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeMismatch& e) {
        g_last_error = e.what();
        return 1;
    } catch (const NonConformantMask& e) {
        g_last_error = e.what();
        return 2;
    } catch (const BadParams& e) {
        g_last_error = e.what();
        return 3;
    } catch (const BadGeometry& e) {
        g_last_error = e.what();
        return 4;
    } catch (const BadMagic& e) {
        g_last_error = e.what();
        return 7;
    } catch (const UnsupportedVersion& e) {
        g_last_error = e.what();
        return 8;
    } catch (const CorruptPayload& e) {
        g_last_error = e.what();
        return 9;
    } catch (const Error& e) {
        g_last_error = e.what();
        return 99;
    }
}

ShflBWMatrix build(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
                   const uint32_t* group_ncols, const uint32_t* cols, const float* values) {
    ShflBWMatrix a;
    a.core.rows = M;
    a.core.cols = K;
    a.core.vector_size = V;
    const uint32_t G = V ? M / V : 0;
    a.core.groups.resize(G);
    size_t off = 0;
    for (uint32_t g = 0; g < G; ++g) {
        auto& grp = a.core.groups[g];
        grp.cols.assign(cols + off, cols + off + group_ncols[g]);
        grp.values.assign(values + off * V, values + (off + group_ncols[g]) * V);
        off += group_ncols[g];
    }
    a.row_indices.assign(row_indices, row_indices + M);
    return a;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

void* ref_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* g) { delete static_cast<std::mt19937_64*>(g); }
uint64_t ref_rng_next(void* g) { return (*static_cast<std::mt19937_64*>(g))(); }

void ref_random_dense(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
    const auto m = random_dense(rows, cols, seed);
    std::memcpy(out, m.values.data(), sizeof(float) * m.values.size());
}

void ref_fill_uniform(void* g, size_t n, float lo, float hi, float* out) {
    auto& rng = *static_cast<std::mt19937_64*>(g);
    for (size_t i = 0; i < n; ++i) out[i] = uniform_float(rng, lo, hi);
}

void ref_random_shflbw_mask(uint32_t m, uint32_t k, uint32_t v, uint32_t cpg, void* g,
                            uint8_t* out) {
    const auto mask = test::random_shflbw_mask(m, k, v, cpg, *static_cast<std::mt19937_64*>(g));
    std::memcpy(out, mask.bits.data(), mask.bits.size());
}

int ref_validate_shflbw(const uint8_t* mask, uint32_t M, uint32_t K, uint32_t V, int* pass,
                        uint32_t* fail_row) {
    return guarded([&] {
        SparsityMask m(M, K, std::vector<uint8_t>(mask, mask + size_t(M) * K));
        const auto rep = validate_pattern(m, PatternKind::ShflBW, {.v = V});
        *pass = rep.pass ? 1 : 0;
        *fail_row = rep.fail_row;
    });
}

// cols / values must hold M*K entries.
int ref_compress(const float* dense, uint32_t dM, uint32_t dK, const uint8_t* mask, uint32_t M,
                 uint32_t K, uint32_t V, uint32_t* row_indices, uint32_t* group_ncols,
                 uint32_t* cols, float* values) {
    return guarded([&] {
        DenseMatrix d(dM, dK, std::vector<float>(dense, dense + size_t(dM) * dK));
        SparsityMask m(M, K, std::vector<uint8_t>(mask, mask + size_t(M) * K));
        const auto sb = compress_shflbw(d, m, V);
        size_t off = 0;
        for (size_t g = 0; g < sb.core.groups.size(); ++g) {
            const auto& grp = sb.core.groups[g];
            group_ncols[g] = uint32_t(grp.cols.size());
            std::memcpy(cols + off, grp.cols.data(), sizeof(uint32_t) * grp.cols.size());
            std::memcpy(values + off * V, grp.values.data(), sizeof(float) * grp.values.size());
            off += grp.cols.size();
        }
        std::memcpy(row_indices, sb.row_indices.data(), sizeof(uint32_t) * sb.row_indices.size());
    });
}

int ref_spmm(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
             const uint32_t* group_ncols, const uint32_t* cols, const float* values,
             const float* B, uint32_t B_rows, uint32_t N, uint32_t t_n, uint32_t t_k,
             unsigned threads, float* C) {
    return guarded([&] {
        const auto a = build(M, K, V, row_indices, group_ncols, cols, values);
        DenseMatrix b(B_rows, N, std::vector<float>(B, B + size_t(B_rows) * N));
        TileConfig cfg;
        if (t_n) cfg.t_n = t_n;
        if (t_k) cfg.t_k = t_k;
        const auto c = spmm_execute(a, b, cfg, threads);
        std::memcpy(C, c.values.data(), sizeof(float) * c.values.size());
    });
}

// Same call on a prebuilt matrix, so timing excludes the flat->struct copy.
void* ref_matrix_new(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
                     const uint32_t* group_ncols, const uint32_t* cols, const float* values) {
    return new ShflBWMatrix(build(M, K, V, row_indices, group_ncols, cols, values));
}
void ref_matrix_free(void* a) { delete static_cast<ShflBWMatrix*>(a); }
void* ref_dense_new(uint32_t rows, uint32_t cols, const float* v) {
    return new DenseMatrix(rows, cols, std::vector<float>(v, v + size_t(rows) * cols));
}
void ref_dense_free(void* d) { delete static_cast<DenseMatrix*>(d); }
int ref_spmm_prebuilt(const void* a, const void* b, unsigned threads, float* C) {
    return guarded([&] {
        const auto c = spmm_execute(*static_cast<const ShflBWMatrix*>(a),
                                    *static_cast<const DenseMatrix*>(b), TileConfig{}, threads);
        if (C) std::memcpy(C, c.values.data(), sizeof(float) * c.values.size());
    });
}

int ref_spmm_dense(const float* A, uint32_t M, uint32_t K, const float* B, uint32_t N, float* C) {
    return guarded([&] {
        DenseMatrix a(M, K, std::vector<float>(A, A + size_t(M) * K));
        DenseMatrix b(K, N, std::vector<float>(B, B + size_t(K) * N));
        const auto c = spmm_dense_oracle(a, b);
        std::memcpy(C, c.values.data(), sizeof(float) * c.values.size());
    });
}

int ref_decompress(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
                   const uint32_t* group_ncols, const uint32_t* cols, const float* values,
                   float* dense) {
    return guarded([&] {
        const auto d = decompress(build(M, K, V, row_indices, group_ncols, cols, values));
        std::memcpy(dense, d.values.data(), sizeof(float) * d.values.size());
    });
}

int ref_conv_output_size(uint32_t H, uint32_t W, uint32_t R, uint32_t S, uint32_t stride,
                         uint32_t pad, uint32_t* P, uint32_t* Q) {
    return guarded([&] {
        const auto pq = conv_output_size(Tensor4(1, H, W, 1), ConvGeometry{R, S, stride, pad});
        *P = pq.first;
        *Q = pq.second;
    });
}

int ref_conv2d(uint32_t Kf, uint32_t Kcols, uint32_t V, const uint32_t* row_indices,
               const uint32_t* group_ncols, const uint32_t* cols, const float* values,
               const float* input, uint32_t C, uint32_t H, uint32_t W, uint32_t Nb, uint32_t R,
               uint32_t S, uint32_t stride, uint32_t pad, unsigned threads, float* out) {
    return guarded([&] {
        const auto w = build(Kf, Kcols, V, row_indices, group_ncols, cols, values);
        Tensor4 in(C, H, W, Nb);
        std::memcpy(in.values.data(), input, sizeof(float) * in.values.size());
        const auto o = conv2d(w, in, ConvGeometry{R, S, stride, pad}, TileConfig{}, threads);
        std::memcpy(out, o.values.data(), sizeof(float) * o.values.size());
    });
}

int ref_stitch_to_blockwise(uint32_t K, uint32_t V, uint32_t G, const uint32_t* group_ncols,
                            const uint32_t* cols, const float* values, uint32_t tile_width,
                            uint32_t* tile_cols, float* tile_vals, uint32_t* tile_group,
                            int* ntiles) {
    return guarded([&] {
        VectorWiseMatrix vw;
        vw.rows = G * V;
        vw.cols = K;
        vw.vector_size = V;
        vw.groups.resize(G);
        size_t off = 0;
        for (uint32_t g = 0; g < G; ++g) {
            vw.groups[g].cols.assign(cols + off, cols + off + group_ncols[g]);
            vw.groups[g].values.assign(values + off * V, values + (off + group_ncols[g]) * V);
            off += group_ncols[g];
        }
        const auto t = stitch_to_blockwise(vw, tile_width);
        int n = 0;
        for (uint32_t g = 0; g < G; ++g)
            for (const auto& tile : t.groups[g]) {
                std::memcpy(tile_cols + size_t(n) * tile_width, tile.cols.data(),
                            sizeof(uint32_t) * tile_width);
                std::memcpy(tile_vals + size_t(n) * tile_width * V, tile.values.data(),
                            sizeof(float) * tile.values.size());
                tile_group[n++] = g;
            }
        *ntiles = n;
    });
}

// SMX1 container (src/container.cpp): encode a kind-3 (Shfl-BW) matrix;
// *size = byte count, bytes copied when out != NULL and cap suffices.
int ref_smx1_encode_shflbw(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
                           const uint32_t* group_ncols, const uint32_t* cols, const float* values, uint8_t* out,
                           size_t cap, size_t* size) {
    return guarded([&] {
        const auto bytes = encode_container(AnyMatrix(build(M, K, V, row_indices, group_ncols, cols, values)));
        *size = bytes.size();
        if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
    });
}

// decode_container + as_shflbw: hdr = {M, K, V, G, total columns}; the arrays
// are filled when non-NULL (sized from a first call with NULLs).
int ref_smx1_decode_shflbw(const uint8_t* bytes, size_t n, uint32_t* hdr, uint32_t* row_indices,
                           uint32_t* group_ncols, uint32_t* cols, float* values) {
    return guarded([&] {
        const auto any = decode_container(std::vector<uint8_t>(bytes, bytes + n));
        const ShflBWMatrix& a = as_shflbw(any);
        const uint32_t V = a.core.vector_size, G = static_cast<uint32_t>(a.core.groups.size());
        size_t total = 0;
        for (const auto& g : a.core.groups) total += g.cols.size();
        hdr[0] = a.core.rows;
        hdr[1] = a.core.cols;
        hdr[2] = V;
        hdr[3] = G;
        hdr[4] = static_cast<uint32_t>(total);
        if (!row_indices) return;
        std::memcpy(row_indices, a.row_indices.data(), sizeof(uint32_t) * a.row_indices.size());
        size_t off = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const auto& grp = a.core.groups[g];
            group_ncols[g] = static_cast<uint32_t>(grp.cols.size());
            std::memcpy(cols + off, grp.cols.data(), sizeof(uint32_t) * grp.cols.size());
            std::memcpy(values + off * V, grp.values.data(), sizeof(float) * grp.values.size());
            off += grp.cols.size();
        }
    });
}

// a valid kind-0 (dense) container, for the kind-mismatch case
int ref_smx1_encode_dense(uint32_t rows, uint32_t cols, const float* v, uint8_t* out, size_t cap, size_t* size) {
    return guarded([&] {
        const auto bytes = encode_container(AnyMatrix(DenseMatrix(rows, cols, std::vector<float>(v, v + size_t(rows) * cols))));
        *size = bytes.size();
        if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
    });
}

// ---- pruning (src/pruning.cpp) ----
namespace {
ImportanceMatrix scores_of(const float* s, uint32_t M, uint32_t K) {
    return ImportanceMatrix(M, K, std::vector<float>(s, s + size_t(M) * K));
}
SparsityMask mask_of(const uint8_t* m, uint32_t M, uint32_t K) {
    return SparsityMask(M, K, std::vector<uint8_t>(m, m + size_t(M) * K));
}
PruneConfig cfg_of(double alpha, double beta_factor, uint32_t v, uint32_t iters, uint64_t seed, uint32_t restarts) {
    PruneConfig c;
    c.alpha = alpha;
    c.beta_factor = beta_factor;
    c.v = v;
    c.kmeans_max_iters = iters;
    c.seed = seed;
    c.restarts = restarts;
    return c;
}
}  // namespace

int ref_kept_score(const float* s, const uint8_t* m, uint32_t M, uint32_t K, double* out) {
    return guarded([&] { *out = kept_score(scores_of(s, M, K), mask_of(m, M, K)); });
}
int ref_prune_unstructured(const float* s, uint32_t M, uint32_t K, double ratio, uint8_t* out) {
    return guarded([&] {
        const auto m = prune_unstructured(scores_of(s, M, K), ratio);
        std::memcpy(out, m.bits.data(), m.bits.size());
    });
}
int ref_prune_vectorwise(const float* s, uint32_t M, uint32_t K, uint32_t v, double alpha, uint8_t* out) {
    return guarded([&] {
        const auto m = prune_vectorwise(scores_of(s, M, K), v, alpha);
        std::memcpy(out, m.bits.data(), m.bits.size());
    });
}
int ref_kmeans_row_grouping(const uint8_t* m, const float* s, uint32_t M, uint32_t K, double alpha,
                            double beta_factor, uint32_t v, uint32_t iters, uint64_t seed, uint32_t restarts,
                            uint32_t* order) {
    return guarded([&] {
        const auto o = kmeans_row_grouping(mask_of(m, M, K), v, cfg_of(alpha, beta_factor, v, iters, seed, restarts),
                                           scores_of(s, M, K));
        std::memcpy(order, o.data(), sizeof(uint32_t) * o.size());
    });
}
int ref_prune_shflbw(const float* s, uint32_t M, uint32_t K, double alpha, double beta_factor, uint32_t v,
                     uint32_t iters, uint64_t seed, uint32_t restarts, uint8_t* mask, uint32_t* perm, double* kept) {
    return guarded([&] {
        const auto r = prune_shflbw(scores_of(s, M, K), cfg_of(alpha, beta_factor, v, iters, seed, restarts));
        std::memcpy(mask, r.mask.bits.data(), r.mask.bits.size());
        std::memcpy(perm, r.permutation.data(), sizeof(uint32_t) * r.permutation.size());
        *kept = r.kept_score;
    });
}

}  // extern "C"

// shflbw/shflbw.hpp -- the reference-compatible C++ API of the B200 library.
//
// Declares, in namespace shflbw, the same types and functions as the
// reference headers (/root/reference/proj/include/shflbw/{errors,matrix,
// formats,spmm,rng}.hpp), so code written against the reference (its unit
// tests, its CLI) compiles and links against libshflbw_b200.so unchanged.
// The per-name forwarding headers (errors.hpp, matrix.hpp, formats.hpp,
// spmm.hpp, rng.hpp) include this file.
//
// What changes behind the same signatures:
//   * compress_shflbw / validate_pattern(ShflBW) / decompress run on the GPU
//     (csrc/convert.cu); spmm_execute / conv2d run the sm_100a kernels
//     (csrc/spmm_sm100.cu, csrc/spmm_simt.cu).  `threads` is accepted and
//     ignored; TileConfig is validated exactly as before.
//   * Arithmetic: by default (SHFLBW_DEVICE_DTYPE unset or f32) the exact
//     CUDA-core kernel -- products rounded then added in ascending k, so
//     results are bit-identical to the reference.  SHFLBW_DEVICE_DTYPE=bf16
//     or f16 rounds operands to 16 bits and runs the tcgen05 tensor-core
//     kernel (fp32 accumulation, within the reference's 1e-5 relative
//     Frobenius --check bar on 16-bit-exact inputs); see DESIGN.md.
//   * spmm_dense_oracle / stitch_tile / tile_mma also run on the device, in
//     the reference's pinned order (mul then add, ascending k).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>
#include <random>

namespace shflbw {

// ---- errors (reference errors.hpp:9-40) -----------------------------------
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShapeMismatch : Error { using Error::Error; };
struct NonConformantMask : Error { using Error::Error; };
struct BadParams : Error { using Error::Error; };
struct BadGeometry : Error { using Error::Error; };
struct BadMagic : Error { using Error::Error; };
struct UnsupportedVersion : Error { using Error::Error; };
struct CorruptPayload : Error { using Error::Error; };

// ---- dense matrix and mask (reference matrix.hpp:14-75) ---------------------
struct DenseMatrix {
    std::uint32_t rows = 0;
    std::uint32_t cols = 0;
    std::vector<float> values;  // row-major

    DenseMatrix() = default;
    DenseMatrix(std::uint32_t r, std::uint32_t c) : rows(r), cols(c), values(std::size_t(r) * c, 0.0f) {}
    DenseMatrix(std::uint32_t r, std::uint32_t c, std::vector<float> v);  // BadParams on bad length / non-finite

    std::size_t size() const { return std::size_t(rows) * cols; }
    float at(std::uint32_t r, std::uint32_t c) const { return values[std::size_t(r) * cols + c]; }
    float& at(std::uint32_t r, std::uint32_t c) { return values[std::size_t(r) * cols + c]; }
    std::span<const float> row(std::uint32_t r) const { return {values.data() + std::size_t(r) * cols, cols}; }
    bool operator==(const DenseMatrix&) const = default;
};

struct SparsityMask {
    std::uint32_t rows = 0;
    std::uint32_t cols = 0;
    std::vector<std::uint8_t> bits;  // row-major, 0 or 1

    SparsityMask() = default;
    SparsityMask(std::uint32_t r, std::uint32_t c) : rows(r), cols(c), bits(std::size_t(r) * c, 0) {}
    SparsityMask(std::uint32_t r, std::uint32_t c, std::vector<std::uint8_t> b);  // BadParams

    std::size_t size() const { return std::size_t(rows) * cols; }
    std::uint8_t at(std::uint32_t r, std::uint32_t c) const { return bits[std::size_t(r) * cols + c]; }
    std::uint8_t& at(std::uint32_t r, std::uint32_t c) { return bits[std::size_t(r) * cols + c]; }
    std::size_t popcount() const;
    double density() const;
    bool operator==(const SparsityMask&) const = default;
};

DenseMatrix apply_mask(const DenseMatrix& dense, const SparsityMask& mask);

// ---- sparse formats (reference formats.hpp:13-124) --------------------------
struct VectorWiseGroup {
    std::vector<std::uint32_t> cols;  // strictly increasing
    std::vector<float> values;        // column-major V x cols.size(): values[j*V + v]
};

struct VectorWiseMatrix {
    std::uint32_t rows = 0;
    std::uint32_t cols = 0;
    std::uint32_t vector_size = 1;
    std::vector<VectorWiseGroup> groups;

    std::uint32_t group_count() const { return static_cast<std::uint32_t>(groups.size()); }
    float value(std::uint32_t g, std::uint32_t v, std::uint32_t j) const {
        return groups[g].values[std::size_t(j) * vector_size + v];
    }
};

struct ShflBWMatrix {
    VectorWiseMatrix core;
    std::vector<std::uint32_t> row_indices;  // compressed row r -> original row
};

struct BlockWiseMatrix {
    std::uint32_t rows = 0;
    std::uint32_t cols = 0;
    std::uint32_t block_size = 1;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> block_coords;
    std::vector<float> block_values;  // row-major V x V per block

    std::uint32_t block_count() const { return static_cast<std::uint32_t>(block_coords.size()); }
};

enum class PatternKind { Unstructured, VectorWise, BlockWise, ShflBW, Balanced };

std::string_view pattern_name(PatternKind kind);
PatternKind parse_pattern(std::string_view name);

struct PatternParams {
    std::uint32_t v = 0;
    std::uint32_t n = 0;
    std::uint32_t m = 0;
};

struct ValidationReport {
    bool pass = true;
    std::uint32_t fail_row = 0;
    std::uint32_t fail_col = 0;
    std::string reason;
};

ValidationReport validate_pattern(const SparsityMask& mask, PatternKind pattern, const PatternParams& params);
ShflBWMatrix compress_shflbw(const DenseMatrix& dense, const SparsityMask& mask, std::uint32_t v);
DenseMatrix decompress(const VectorWiseMatrix& m);
DenseMatrix decompress(const ShflBWMatrix& m);
DenseMatrix decompress(const BlockWiseMatrix& m);

inline constexpr std::uint32_t kPadColumn = 0xffffffffu;

struct StitchedTile {
    std::vector<std::uint32_t> cols;  // tile_width entries, kPadColumn = padding
    std::vector<float> values;        // column-major V x tile_width
    std::uint32_t pad_cols = 0;
};

struct GroupTiling {
    std::uint32_t vector_size = 1;
    std::uint32_t tile_width = 1;
    std::vector<std::vector<StitchedTile>> groups;
};

GroupTiling stitch_to_blockwise(const VectorWiseMatrix& vw, std::uint32_t tile_width);

// ---- execution (reference spmm.hpp:13-94) -------------------------------------
struct TileConfig {
    std::uint32_t t_m = 64;
    std::uint32_t t_n = 16;
    std::uint32_t t_k = 8;
    std::uint32_t regfile_size = 4096;
    std::uint32_t pipe_stage = 2;
    std::uint32_t meta_prefetch_stage = 4;

    void validate() const;  // BadParams
};

DenseMatrix spmm_execute(const ShflBWMatrix& a, const DenseMatrix& b, const TileConfig& cfg,
                         unsigned threads = 1);
DenseMatrix spmm_dense_oracle(const DenseMatrix& a_dense, const DenseMatrix& b);
std::vector<float> stitch_tile(const std::vector<std::uint32_t>& group_cols, std::size_t chunk_begin,
                               std::size_t t_k, const DenseMatrix& b, std::size_t slice_begin,
                               std::size_t t_n);
void tile_mma(std::span<float> acc, std::span<const float> a_tile, std::span<const float> b_tile,
              std::size_t v_rows, std::size_t k_len, std::size_t t_n);
double relative_frobenius_error(const DenseMatrix& x, const DenseMatrix& y);

struct Tensor4 {
    std::uint32_t c = 0, h = 0, w = 0, n = 0;
    std::vector<float> values;  // [c][h][w][n]

    Tensor4() = default;
    Tensor4(std::uint32_t c_, std::uint32_t h_, std::uint32_t w_, std::uint32_t n_)
        : c(c_), h(h_), w(w_), n(n_), values(std::size_t(c_) * h_ * w_ * n_, 0.0f) {}
    std::size_t size() const { return values.size(); }
    float at(std::uint32_t ci, std::uint32_t hi, std::uint32_t wi, std::uint32_t ni) const {
        return values[((std::size_t(ci) * h + hi) * w + wi) * n + ni];
    }
    float& at(std::uint32_t ci, std::uint32_t hi, std::uint32_t wi, std::uint32_t ni) {
        return values[((std::size_t(ci) * h + hi) * w + wi) * n + ni];
    }
};

struct ConvGeometry {
    std::uint32_t r = 1, s = 1;
    std::uint32_t stride = 1;
    std::uint32_t pad = 0;
};

Tensor4 conv2d(const ShflBWMatrix& weights, const Tensor4& input, const ConvGeometry& geo,
               const TileConfig& cfg, unsigned threads = 1);
std::pair<std::uint32_t, std::uint32_t> conv_output_size(const Tensor4& input, const ConvGeometry& geo);

// ---- synthetic inputs (reference rng.hpp:14-24) --------------------------------
inline double uniform01(std::mt19937_64& rng) { return double(rng() >> 11) * 0x1.0p-53; }
inline float uniform_float(std::mt19937_64& rng, float lo, float hi) {
    return lo + float(uniform01(rng)) * (hi - lo);
}
DenseMatrix random_dense(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed);

}  // namespace shflbw

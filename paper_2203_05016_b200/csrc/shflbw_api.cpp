// shflbw_api.cpp -- the reference-compatible C++ API (include/shflbw/shflbw.hpp)
// implemented over the C ABI (include/shflbw_cu.h).
//
// Value semantics are the reference's (include/shflbw/matrix.hpp:12-13):
// inputs by const reference, outputs by value in host std::vectors.  Each
// call therefore copies its operands host->device on this thread's
// per-thread stream, runs the device kernels, and copies the result back.
// Code that wants device-resident weights and no copies uses the C ABI (or
// the Python mirror) directly.
//
// Host-side code here is limited to argument validation with the
// reference's exception classes, layout marshalling of the host structs, and
// the out-of-scope pattern utilities (vector-/block-wise/balanced validators,
// block-wise decompress, stitch_to_blockwise) that only the pruning side of
// the reference uses.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>

#include "shflbw/shflbw.hpp"
#include "shflbw_cu.h"

namespace sbw {
void retain_pool();  // convert.cu: keep the pool's memory across synchronisations
}

namespace shflbw {
namespace {

cudaStream_t stream() { return cudaStreamPerThread; }
shflbw_stream_t sstream() { return reinterpret_cast<shflbw_stream_t>(cudaStreamPerThread); }

[[noreturn]] void raise(int status, const std::string& where) {
    const std::string msg = where + ": " + shflbw_cu_last_error();
    switch (status) {
        case SHFLBW_SHAPE_MISMATCH: throw ShapeMismatch(msg);
        case SHFLBW_NONCONFORMANT_MASK: throw NonConformantMask(msg);
        case SHFLBW_BAD_PARAMS: throw BadParams(msg);
        case SHFLBW_BAD_GEOMETRY: throw BadGeometry(msg);
        case SHFLBW_BAD_MAGIC: throw BadMagic(msg);
        case SHFLBW_UNSUPPORTED_VERSION: throw UnsupportedVersion(msg);
        case SHFLBW_CORRUPT_PAYLOAD: throw CorruptPayload(msg);
        default: throw Error(msg);
    }
}

void check(int status, const char* where) {
    if (status != SHFLBW_OK) raise(status, where);
}

void check_cuda(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw Error(std::string(where) + ": " + cudaGetErrorString(e));
}

// device value type used for SpMM / conv operands.  Default f32: the exact
// CUDA-core path, bit-identical to the reference (its unit tests pass
// unchanged).  SHFLBW_DEVICE_DTYPE=bf16|f16 selects the tcgen05 tensor-core
// path (operands rounded to 16 bits, fp32 accumulation).
int compute_dtype() {
    static const int dt = [] {
        const char* e = std::getenv("SHFLBW_DEVICE_DTYPE");
        if (e && (!std::strcmp(e, "f16") || !std::strcmp(e, "fp16"))) return static_cast<int>(SHFLBW_F16);
        if (e && !std::strcmp(e, "bf16")) return static_cast<int>(SHFLBW_BF16);
        return static_cast<int>(SHFLBW_F32);
    }();
    return dt;
}
int dtype_size(int dt) { return dt == SHFLBW_F32 ? 4 : 2; }

// Scratch from the device's stream-ordered pool on this thread's stream (a
// plain cudaMalloc / cudaFree per call synchronises the device).
struct DeviceBuffer {
    void* p = nullptr;
    explicit DeviceBuffer(size_t bytes) {
        sbw::retain_pool();
        check_cuda(cudaMallocAsync(&p, bytes ? bytes : 16, stream()), "cudaMallocAsync");
    }
    ~DeviceBuffer() {
        if (p) cudaFreeAsync(p, stream());
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct DeviceMatrix {
    shflbw_cu_matrix m{};
    ~DeviceMatrix() { shflbw_cu_matrix_free(&m); }
};

void upload_host(const void* src, DeviceBuffer& dst, size_t bytes) {
    if (bytes) check_cuda(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyHostToDevice, stream()), "H2D");
}

// host ShflBWMatrix -> device layout (values rounded to `dtype`)
void upload_matrix(const ShflBWMatrix& a, int dtype, DeviceMatrix& out) {
    const auto& core = a.core;
    const uint32_t V = core.vector_size;
    if (V == 0 || core.rows % V != 0 || core.group_count() != core.rows / V)
        throw BadParams("ShflBWMatrix: group count must equal M / V");
    std::vector<uint32_t> ncols(core.group_count()), cols;
    std::vector<float> vals;
    size_t total = 0;
    for (const auto& g : core.groups) total += g.cols.size();
    cols.reserve(total);
    vals.reserve(total * V);
    for (uint32_t g = 0; g < core.group_count(); ++g) {
        const auto& grp = core.groups[g];
        if (grp.values.size() != grp.cols.size() * V) throw BadParams("group values size != V * n_g");
        ncols[g] = static_cast<uint32_t>(grp.cols.size());
        cols.insert(cols.end(), grp.cols.begin(), grp.cols.end());
        vals.insert(vals.end(), grp.values.begin(), grp.values.end());
    }
    check(shflbw_cu_matrix_upload(static_cast<int32_t>(core.rows), static_cast<int32_t>(core.cols),
                                  static_cast<int32_t>(V), a.row_indices.data(), ncols.data(), cols.data(),
                                  vals.data(), dtype, &out.m, sstream()),
          "upload");
}

// host f32 -> device 16-bit with a 16-byte aligned row stride
struct DeviceOperand {
    std::unique_ptr<DeviceBuffer> buf;
    int64_t ld = 0;
};

DeviceOperand upload_operand(const float* src, size_t rows, size_t cols, int dtype) {
    DeviceOperand op;
    op.ld = static_cast<int64_t>((cols + 7) / 8 * 8);
    DeviceBuffer staging(rows * cols * sizeof(float));
    upload_host(src, staging, rows * cols * sizeof(float));
    op.buf = std::make_unique<DeviceBuffer>(rows * op.ld * dtype_size(dtype));
    if (rows && cols) {
        if (static_cast<size_t>(op.ld) == cols) {
            check(shflbw_cu_convert(staging.p, SHFLBW_F32, op.buf->p, dtype, static_cast<int64_t>(rows * cols),
                                    sstream()),
                  "convert");
        } else {  // one pitched convert into the 16-byte aligned rows
            check_cuda(cudaMemsetAsync(op.buf->p, 0, rows * op.ld * dtype_size(dtype), stream()), "memset");
            check(shflbw_cu_convert_2d(staging.p, SHFLBW_F32, static_cast<int64_t>(cols), op.buf->p, dtype, op.ld,
                                       static_cast<int64_t>(rows), static_cast<int64_t>(cols), sstream()),
                  "convert");
        }
    }
    check_cuda(cudaStreamSynchronize(stream()), "sync");
    return op;
}

void check_row_indices(const ShflBWMatrix& a, bool conv) {
    auto bad = [&](const char* msg) {
        if (conv) throw BadGeometry(msg);
        throw ShapeMismatch(msg);
    };
    if (a.row_indices.size() != a.core.rows) bad("row_indices length != M");
    for (uint32_t r : a.row_indices)
        if (r >= a.core.rows) bad("row index out of range");
}

}  // namespace

// ---------------------------------------------------------------- matrix.hpp

DenseMatrix::DenseMatrix(std::uint32_t r, std::uint32_t c, std::vector<float> v)
    : rows(r), cols(c), values(std::move(v)) {
    if (values.size() != std::size_t(rows) * cols) throw BadParams("DenseMatrix: values length != rows * cols");
    for (float x : values)
        if (!std::isfinite(x)) throw BadParams("DenseMatrix: non-finite value");
}

SparsityMask::SparsityMask(std::uint32_t r, std::uint32_t c, std::vector<std::uint8_t> b)
    : rows(r), cols(c), bits(std::move(b)) {
    if (bits.size() != std::size_t(rows) * cols) throw BadParams("SparsityMask: bits length != rows * cols");
    for (std::uint8_t x : bits)
        if (x > 1) throw BadParams("SparsityMask: entries must be 0 or 1");
}

std::size_t SparsityMask::popcount() const {
    return static_cast<std::size_t>(std::count(bits.begin(), bits.end(), std::uint8_t{1}));
}

double SparsityMask::density() const { return bits.empty() ? 0.0 : double(popcount()) / double(size()); }

DenseMatrix apply_mask(const DenseMatrix& dense, const SparsityMask& mask) {
    if (dense.rows != mask.rows || dense.cols != mask.cols)
        throw ShapeMismatch("apply_mask: dense and mask shapes differ");
    DenseMatrix out(dense.rows, dense.cols);
    for (std::size_t i = 0; i < out.values.size(); ++i) out.values[i] = mask.bits[i] ? dense.values[i] : 0.0f;
    return out;
}

DenseMatrix random_dense(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    DenseMatrix m(rows, cols);
    for (auto& x : m.values) x = uniform_float(rng, -1.0f, 1.0f);
    return m;
}

// ---------------------------------------------------------------- formats.hpp

std::string_view pattern_name(PatternKind kind) {
    switch (kind) {
        case PatternKind::Unstructured: return "unstructured";
        case PatternKind::VectorWise: return "vector_wise";
        case PatternKind::BlockWise: return "block_wise";
        case PatternKind::ShflBW: return "shfl_bw";
        case PatternKind::Balanced: return "balanced";
    }
    return "?";
}

PatternKind parse_pattern(std::string_view name) {
    if (name == "unstructured") return PatternKind::Unstructured;
    if (name == "vector_wise" || name == "vw") return PatternKind::VectorWise;
    if (name == "block_wise" || name == "bw") return PatternKind::BlockWise;
    if (name == "shfl_bw" || name == "shflbw") return PatternKind::ShflBW;
    if (name == "balanced") return PatternKind::Balanced;
    throw BadParams("unknown pattern: " + std::string(name));
}

namespace {

ValidationReport failed(std::uint32_t r, std::uint32_t c, std::string why) {
    ValidationReport rep;
    rep.pass = false;
    rep.fail_row = r;
    rep.fail_col = c;
    rep.reason = std::move(why);
    return rep;
}

}  // namespace

ValidationReport validate_pattern(const SparsityMask& mask, PatternKind pattern, const PatternParams& params) {
    const uint32_t M = mask.rows, K = mask.cols;
    switch (pattern) {
        case PatternKind::Unstructured:
            return {};
        case PatternKind::ShflBW: {
            if (params.v == 0 || M % params.v != 0) throw BadParams("V must divide M");
            DeviceBuffer d(mask.bits.size());
            upload_host(mask.bits.data(), d, mask.bits.size());
            int32_t pass = 1;
            uint32_t fail_row = 0;
            check(shflbw_cu_validate(d.as<uint8_t>(), M, K, params.v, &pass, &fail_row, sstream()),
                  "validate_pattern");
            if (pass) return {};
            return failed(fail_row, 0, "support class size is not a multiple of V");
        }
        case PatternKind::VectorWise: {  // pruning-side utility (host)
            if (params.v == 0 || M % params.v != 0) throw BadParams("V must divide M");
            for (uint32_t lead = 0; lead < M; lead += params.v)
                for (uint32_t r = lead + 1; r < lead + params.v; ++r)
                    for (uint32_t c = 0; c < K; ++c)
                        if (mask.at(r, c) != mask.at(lead, c)) return failed(r, c, "row support differs from group leader");
            return {};
        }
        case PatternKind::BlockWise: {  // pruning-side utility (host)
            const uint32_t v = params.v;
            if (v == 0 || M % v != 0 || K % v != 0) throw BadParams("V must divide both M and K");
            for (uint32_t br = 0; br < M; br += v)
                for (uint32_t bc = 0; bc < K; bc += v)
                    for (uint32_t i = 0; i < v; ++i)
                        for (uint32_t j = 0; j < v; ++j)
                            if (mask.at(br + i, bc + j) != mask.at(br, bc))
                                return failed(br + i, bc + j, "block is neither kept nor pruned as a whole");
            return {};
        }
        case PatternKind::Balanced: {  // pruning-side utility (host)
            if (params.m == 0 || params.n > params.m || K % params.m != 0)
                throw BadParams("balanced pattern needs n <= m and m | K");
            for (uint32_t r = 0; r < M; ++r)
                for (uint32_t w = 0; w < K; w += params.m) {
                    uint32_t cnt = 0;
                    for (uint32_t j = 0; j < params.m; ++j) cnt += mask.at(r, w + j);
                    if (cnt != params.n)
                        return failed(r, w, "window holds " + std::to_string(cnt) + " non-zeros, expected " +
                                                std::to_string(params.n));
                }
            return {};
        }
    }
    throw BadParams("unknown pattern kind");
}

ShflBWMatrix compress_shflbw(const DenseMatrix& dense, const SparsityMask& mask, std::uint32_t v) {
    if (dense.rows != mask.rows || dense.cols != mask.cols)
        throw ShapeMismatch("compress_shflbw: dense and mask shapes differ");
    const uint32_t M = mask.rows, K = mask.cols;
    DeviceBuffer dd(dense.values.size() * sizeof(float)), dm(mask.bits.size());
    upload_host(dense.values.data(), dd, dense.values.size() * sizeof(float));
    upload_host(mask.bits.data(), dm, mask.bits.size());
    DeviceMatrix out;
    uint32_t fail_row = 0;
    // F32 storage: the host result keeps the weights bit-exact, like the reference
    check(shflbw_cu_compress(dd.p, SHFLBW_F32, dm.as<uint8_t>(), M, K, v, SHFLBW_F32, &out.m, &fail_row, sstream()),
          "compress_shflbw");
    const uint32_t G = M / v;
    ShflBWMatrix res;
    res.core.rows = M;
    res.core.cols = K;
    res.core.vector_size = v;
    res.row_indices.resize(M);
    std::vector<uint32_t> ncols(G), cols(static_cast<size_t>(out.m.total_cols) + 1);
    std::vector<float> vals(static_cast<size_t>(out.m.total_cols) * v + 1);
    check(shflbw_cu_matrix_download(&out.m, res.row_indices.data(), ncols.data(), cols.data(), vals.data(),
                                    sstream()),
          "compress_shflbw");
    res.core.groups.resize(G);
    size_t off = 0;
    for (uint32_t g = 0; g < G; ++g) {
        auto& grp = res.core.groups[g];
        grp.cols.assign(cols.begin() + off, cols.begin() + off + ncols[g]);
        grp.values.assign(vals.begin() + off * v, vals.begin() + (off + ncols[g]) * v);
        off += ncols[g];
    }
    return res;
}

DenseMatrix decompress(const ShflBWMatrix& m) {
    DeviceMatrix dm;
    upload_matrix(m, SHFLBW_F32, dm);
    DenseMatrix out(m.core.rows, m.core.cols);
    DeviceBuffer d(out.values.size() * sizeof(float));
    check(shflbw_cu_decompress(&dm.m, d.as<float>(), sstream()), "decompress");
    if (!out.values.empty())
        check_cuda(cudaMemcpyAsync(out.values.data(), d.p, out.values.size() * sizeof(float), cudaMemcpyDeviceToHost,
                                   stream()),
                   "D2H");
    check_cuda(cudaStreamSynchronize(stream()), "sync");
    return out;
}

DenseMatrix decompress(const VectorWiseMatrix& m) {
    ShflBWMatrix s;
    s.core = m;
    s.row_indices.resize(m.rows);
    for (uint32_t r = 0; r < m.rows; ++r) s.row_indices[r] = r;
    return decompress(s);
}

DenseMatrix decompress(const BlockWiseMatrix& m) {  // block-wise comparator format (host layout utility)
    DenseMatrix out(m.rows, m.cols);
    const uint32_t v = m.block_size;
    for (uint32_t b = 0; b < m.block_count(); ++b) {
        const auto [br, bc] = m.block_coords[b];
        for (uint32_t i = 0; i < v; ++i)
            for (uint32_t j = 0; j < v; ++j)
                out.at(br * v + i, bc * v + j) = m.block_values[(std::size_t(b) * v + i) * v + j];
    }
    return out;
}

GroupTiling stitch_to_blockwise(const VectorWiseMatrix& vw, std::uint32_t tile_width) {
    // layout utility (host): the device format applies the same padding rule
    // with tile_width = SHFLBW_K_TILE inside the converter
    if (tile_width == 0) throw BadParams("tile_width must be positive");
    const uint32_t v = vw.vector_size;
    GroupTiling t;
    t.vector_size = v;
    t.tile_width = tile_width;
    for (const auto& grp : vw.groups) {
        std::vector<StitchedTile> tiles;
        for (size_t begin = 0; begin < grp.cols.size(); begin += tile_width) {
            const size_t avail = std::min<size_t>(tile_width, grp.cols.size() - begin);
            StitchedTile tile;
            tile.cols.assign(tile_width, kPadColumn);
            tile.values.assign(size_t(tile_width) * v, 0.0f);
            tile.pad_cols = static_cast<uint32_t>(tile_width - avail);
            std::copy_n(grp.cols.begin() + begin, avail, tile.cols.begin());
            std::copy_n(grp.values.begin() + begin * v, avail * v, tile.values.begin());
            tiles.push_back(std::move(tile));
        }
        t.groups.push_back(std::move(tiles));
    }
    return t;
}

// ---------------------------------------------------------------- spmm.hpp

void TileConfig::validate() const {
    if (t_m == 0 || t_n == 0 || t_k == 0) throw BadParams("tile sizes must be positive");
    if (std::uint64_t(t_m) * t_n > regfile_size) throw BadParams("T_M * T_N exceeds the register-file budget");
    if (pipe_stage < 2) throw BadParams("pipe_stage must be >= 2");
    if (meta_prefetch_stage < 1) throw BadParams("meta_prefetch_stage must be >= 1");
}

DenseMatrix spmm_execute(const ShflBWMatrix& a, const DenseMatrix& b, const TileConfig& cfg, unsigned) {
    cfg.validate();
    if (a.core.cols != b.rows) throw ShapeMismatch("spmm: A columns != B rows");
    check_row_indices(a, false);
    const int dt = compute_dtype();
    DeviceMatrix dm;
    upload_matrix(a, dt, dm);
    DeviceOperand op = upload_operand(b.values.data(), b.rows, b.cols, dt);
    DenseMatrix c(a.core.rows, b.cols);
    DeviceBuffer dc(c.values.size() * sizeof(float));
    check_cuda(cudaMemsetAsync(dc.p, 0, c.values.size() * sizeof(float), stream()), "memset");
    check(shflbw_cu_spmm(&dm.m, op.buf->p, b.rows, b.cols, op.ld, dc.p, SHFLBW_F32, b.cols, sstream()),
          "spmm_execute");
    if (!c.values.empty())
        check_cuda(cudaMemcpyAsync(c.values.data(), dc.p, c.values.size() * sizeof(float), cudaMemcpyDeviceToHost,
                                   stream()),
                   "D2H");
    check_cuda(cudaStreamSynchronize(stream()), "sync");
    return c;
}

DenseMatrix spmm_dense_oracle(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.cols != b.rows) throw ShapeMismatch("oracle: A columns != B rows");
    DenseMatrix c(a.rows, b.cols);
    DeviceBuffer da(a.values.size() * 4), db(b.values.size() * 4), dc(c.values.size() * 4);
    upload_host(a.values.data(), da, a.values.size() * 4);
    upload_host(b.values.data(), db, b.values.size() * 4);
    check(shflbw_cu_dense_matmul_f32(da.as<float>(), a.rows, a.cols, db.as<float>(), b.cols, dc.as<float>(),
                                     sstream()),
          "spmm_dense_oracle");
    if (!c.values.empty())
        check_cuda(cudaMemcpyAsync(c.values.data(), dc.p, c.values.size() * 4, cudaMemcpyDeviceToHost, stream()),
                   "D2H");
    check_cuda(cudaStreamSynchronize(stream()), "sync");
    return c;
}

std::vector<float> stitch_tile(const std::vector<std::uint32_t>& group_cols, std::size_t chunk_begin,
                               std::size_t t_k, const DenseMatrix& b, std::size_t slice_begin, std::size_t t_n) {
    std::vector<float> staging(t_k * t_n, 0.0f);
    if (staging.empty()) return staging;
    DeviceBuffer dcols(group_cols.size() * 4), db(b.values.size() * 4), ds(staging.size() * 4);
    upload_host(group_cols.data(), dcols, group_cols.size() * 4);
    upload_host(b.values.data(), db, b.values.size() * 4);
    check(shflbw_cu_stitch_tile(dcols.as<uint32_t>(), static_cast<int64_t>(group_cols.size()),
                                static_cast<int64_t>(chunk_begin), static_cast<int64_t>(t_k), db.as<float>(),
                                b.rows, b.cols, static_cast<int64_t>(slice_begin), static_cast<int64_t>(t_n),
                                ds.as<float>(), sstream()),
          "stitch_tile");
    check_cuda(cudaMemcpyAsync(staging.data(), ds.p, staging.size() * 4, cudaMemcpyDeviceToHost, stream()), "D2H");
    check_cuda(cudaStreamSynchronize(stream()), "sync");
    return staging;
}

void tile_mma(std::span<float> acc, std::span<const float> a_tile, std::span<const float> b_tile,
              std::size_t v_rows, std::size_t k_len, std::size_t t_n) {
    if (acc.size() < v_rows * t_n || a_tile.size() < k_len * v_rows || b_tile.size() < k_len * t_n)
        throw ShapeMismatch("tile_mma: span sizes do not cover the tile");
    if (v_rows * t_n == 0) return;
    DeviceBuffer dacc(acc.size_bytes()), da(a_tile.size_bytes() + 4), dbt(b_tile.size_bytes() + 4);
    upload_host(acc.data(), dacc, acc.size_bytes());
    upload_host(a_tile.data(), da, a_tile.size_bytes());
    upload_host(b_tile.data(), dbt, b_tile.size_bytes());
    check(shflbw_cu_tile_mma(dacc.as<float>(), da.as<float>(), dbt.as<float>(), static_cast<int64_t>(v_rows),
                             static_cast<int64_t>(k_len), static_cast<int64_t>(t_n), sstream()),
          "tile_mma");
    check_cuda(cudaMemcpyAsync(acc.data(), dacc.p, acc.size_bytes(), cudaMemcpyDeviceToHost, stream()), "D2H");
    check_cuda(cudaStreamSynchronize(stream()), "sync");
}

double relative_frobenius_error(const DenseMatrix& x, const DenseMatrix& y) {
    // the reference's parity metric (src/spmm.cpp:163-175), a checker
    if (x.rows != y.rows || x.cols != y.cols) throw ShapeMismatch("relative_frobenius_error: shapes differ");
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < x.values.size(); ++i) {
        const double d = double(x.values[i]) - double(y.values[i]);
        num += d * d;
        den += double(y.values[i]) * double(y.values[i]);
    }
    if (den == 0.0) return num == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
    return std::sqrt(num) / std::sqrt(den);
}

std::pair<std::uint32_t, std::uint32_t> conv_output_size(const Tensor4& input, const ConvGeometry& geo) {
    if (geo.r == 0 || geo.s == 0 || geo.stride == 0) throw BadGeometry("filter sizes and stride must be positive");
    int32_t P = 0, Q = 0;
    const int st = shflbw_cu_conv_output_size(static_cast<int32_t>(input.h), static_cast<int32_t>(input.w),
                                              static_cast<int32_t>(geo.r), static_cast<int32_t>(geo.s),
                                              static_cast<int32_t>(geo.stride), static_cast<int32_t>(geo.pad), &P, &Q);
    if (st != SHFLBW_OK) raise(st, "conv_output_size");
    return {static_cast<uint32_t>(P), static_cast<uint32_t>(Q)};
}

Tensor4 conv2d(const ShflBWMatrix& weights, const Tensor4& input, const ConvGeometry& geo, const TileConfig& cfg,
               unsigned) {
    cfg.validate();
    const auto [P, Q] = conv_output_size(input, geo);
    if (uint64_t(weights.core.cols) != uint64_t(input.c) * geo.r * geo.s) throw BadGeometry("weight columns != C*R*S");
    check_row_indices(weights, true);
    const int dt = compute_dtype();
    DeviceMatrix dm;
    upload_matrix(weights, dt, dm);
    Tensor4 out(weights.core.rows, P, Q, input.n);
    DeviceBuffer staging(input.values.size() * 4), din(input.values.size() * dtype_size(dt) + 16),
        dout(out.values.size() * 4);
    upload_host(input.values.data(), staging, input.values.size() * 4);
    check(shflbw_cu_convert(staging.p, SHFLBW_F32, din.p, dt, static_cast<int64_t>(input.values.size()), sstream()),
          "convert");
    check_cuda(cudaMemsetAsync(dout.p, 0, out.values.size() * 4, stream()), "memset");
    check(shflbw_cu_conv2d(&dm.m, din.p, input.c, input.h, input.w, input.n, geo.r, geo.s, geo.stride, geo.pad, dout.p,
                           SHFLBW_F32, sstream()),
          "conv2d");
    if (!out.values.empty())
        check_cuda(cudaMemcpyAsync(out.values.data(), dout.p, out.values.size() * 4, cudaMemcpyDeviceToHost, stream()),
                   "D2H");
    check_cuda(cudaStreamSynchronize(stream()), "sync");
    return out;
}

}  // namespace shflbw

// tc_inst_f16_conv.cu -- implicit-GEMM conv kernels of tc_kernels.cuh for f16 operands
// (one translation unit per dtype and operand kind, so nvcc builds them in parallel).
#include "tc_kernels.cuh"

namespace sbw {
namespace tc {
template SBW_TC_DISPATCH(SHFLBW_F16, 1);
}  // namespace tc
}  // namespace sbw

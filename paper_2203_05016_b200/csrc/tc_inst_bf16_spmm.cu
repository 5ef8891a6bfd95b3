// tc_inst_bf16_spmm.cu -- SpMM kernels of tc_kernels.cuh for bf16 operands
// (one translation unit per dtype and operand kind, so nvcc builds them in parallel).
#include "tc_kernels.cuh"

namespace sbw {
namespace tc {
template SBW_TC_DISPATCH(SHFLBW_BF16, 0);
}  // namespace tc
}  // namespace sbw

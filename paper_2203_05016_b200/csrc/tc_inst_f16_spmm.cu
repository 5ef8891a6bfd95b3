// tc_inst_f16_spmm.cu -- SpMM kernels of tc_kernels.cuh for f16 operands
// (one translation unit per dtype and operand kind, so nvcc builds them in parallel).
#include "tc_kernels.cuh"

namespace sbw {
namespace tc {
template SBW_TC_DISPATCH(SHFLBW_F16, 0);
}  // namespace tc
}  // namespace sbw

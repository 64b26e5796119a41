// gemm_tc_mm_bf16.cu -- instantiation of tc_gemm_kernel variants (see gemm_tc.cuh)
#include "gemm_tc.cuh"

namespace xtc {

XTC_TC_VARIANT(false, false, 1, false, 1)
XTC_TC_VARIANT(false, false, 2, false, 1)

}  // namespace xtc

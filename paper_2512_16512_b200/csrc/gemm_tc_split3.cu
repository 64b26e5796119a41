// gemm_tc_split3.cu -- instantiation of tc_gemm_kernel variants (see gemm_tc.cuh)
#include "gemm_tc.cuh"

namespace xtc {

XTC_TC_VARIANT(true, false, 1, true, 1)

}  // namespace xtc

// gemm_tc_ms2.cu -- instantiation of the matmul tc_gemm_kernel variants with two 128-row
// M-subtiles per CTA (tile_m = 256 * cta_group; see gemm_tc.cuh)
#include "gemm_tc.cuh"

namespace xtc {

XTC_TC_VARIANT(false, false, 1, false, 2)
XTC_TC_VARIANT(false, false, 2, false, 2)
XTC_TC_VARIANT(true, false, 1, false, 2)
XTC_TC_VARIANT(true, false, 2, false, 2)

}  // namespace xtc

// gemm_simt_tm2.cu -- instantiation of the SIMT kernel variants with thread-tile height 2
#include "gemm_simt.cuh"

namespace xtc {

XTC_SIMT_TM(2)

}  // namespace xtc

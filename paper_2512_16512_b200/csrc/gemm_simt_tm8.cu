// gemm_simt_tm8.cu -- instantiation of the SIMT kernel variants with thread-tile height 8
#include "gemm_simt.cuh"

namespace xtc {

XTC_SIMT_TM(8)

}  // namespace xtc

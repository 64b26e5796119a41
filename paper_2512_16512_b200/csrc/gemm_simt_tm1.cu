// gemm_simt_tm1.cu -- instantiation of the SIMT kernel variants with thread-tile height 1
#include "gemm_simt.cuh"

namespace xtc {

XTC_SIMT_TM(1)

}  // namespace xtc

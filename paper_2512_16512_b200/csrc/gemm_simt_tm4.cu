// gemm_simt_tm4.cu -- instantiation of the SIMT kernel variants with thread-tile height 4
#include "gemm_simt.cuh"

namespace xtc {

XTC_SIMT_TM(4)

}  // namespace xtc

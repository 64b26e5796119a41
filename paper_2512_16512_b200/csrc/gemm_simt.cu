// gemm_simt.cu -- dispatch of the SIMT fp32 engine (kernel: gemm_simt.cuh)
#include "gemm_simt.cuh"

namespace xtc {

XTC_SIMT_TM_EXTERN(1)
XTC_SIMT_TM_EXTERN(2)
XTC_SIMT_TM_EXTERN(4)
XTC_SIMT_TM_EXTERN(8)

cudaError_t launch_simt_gemm(int tm, int tn, int u, int vec, const SimtParams& p, int grid, int block, int smem,
                             cudaStream_t st) {
    switch (tm) {
        case 1: return launch_simt_n<1>(tn, u, vec, p, grid, block, smem, st);
        case 2: return launch_simt_n<2>(tn, u, vec, p, grid, block, smem, st);
        case 4: return launch_simt_n<4>(tn, u, vec, p, grid, block, smem, st);
        default: return launch_simt_n<8>(tn, u, vec, p, grid, block, smem, st);
    }
}

}  // namespace xtc

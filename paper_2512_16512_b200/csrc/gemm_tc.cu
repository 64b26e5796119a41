// gemm_tc.cu -- dispatch of the tcgen05 GEMM / implicit-GEMM conv variants (the kernel
// is in gemm_tc.cuh; each variant is compiled in its own gemm_tc_*.cu).
#include "gemm_tc.cuh"

namespace xtc {

XTC_TC_EXTERN(false, false, 1, false, 1)
XTC_TC_EXTERN(false, false, 2, false, 1)
XTC_TC_EXTERN(false, true, 1, false, 1)
XTC_TC_EXTERN(false, true, 2, false, 1)
XTC_TC_EXTERN(true, false, 1, false, 1)
XTC_TC_EXTERN(true, false, 2, false, 1)
XTC_TC_EXTERN(true, true, 1, false, 1)
XTC_TC_EXTERN(true, true, 2, false, 1)
XTC_TC_EXTERN(true, false, 1, true, 1)
XTC_TC_EXTERN(false, false, 1, false, 2)
XTC_TC_EXTERN(false, false, 2, false, 2)
XTC_TC_EXTERN(true, false, 1, false, 2)
XTC_TC_EXTERN(true, false, 2, false, 2)

template <int CG>
static cudaError_t launch_tc_cg(bool tf32, bool conv, const CUtensorMap& a, const CUtensorMap& b,
                                const CUtensorMap& c, const TcParams& p, int grid, int smem, cudaStream_t st) {
    if (p.ms == 2)    // two M-subtiles per CTA (matmul only)
        return tf32 ? launch_tc_t<true, false, CG, false, 2>(a, b, c, p, grid, smem, st)
                    : launch_tc_t<false, false, CG, false, 2>(a, b, c, p, grid, smem, st);
    if (tf32) return conv ? launch_tc_t<true, true, CG, false, 1>(a, b, c, p, grid, smem, st)
                          : launch_tc_t<true, false, CG, false, 1>(a, b, c, p, grid, smem, st);
    return conv ? launch_tc_t<false, true, CG, false, 1>(a, b, c, p, grid, smem, st)
                : launch_tc_t<false, false, CG, false, 1>(a, b, c, p, grid, smem, st);
}

cudaError_t launch_tc_gemm(bool tf32, bool conv, int cta_group, const CUtensorMap& a, const CUtensorMap& b,
                           const CUtensorMap& c, const TcParams& p, int grid, int smem, cudaStream_t st) {
    if (p.lo_off) return launch_tc_t<true, false, 1, true, 1>(a, b, c, p, grid, smem, st);   // 3xTF32 split (fp32)
    if (cta_group == 2) return launch_tc_cg<2>(tf32, conv, a, b, c, p, grid, smem, st);
    return launch_tc_cg<1>(tf32, conv, a, b, c, p, grid, smem, st);
}

}  // namespace xtc

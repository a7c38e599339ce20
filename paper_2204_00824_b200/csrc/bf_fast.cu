// Instantiations of bf_fast_kernel (own translation unit: compiled in parallel with
// tsdg_gpu.cu).  Tuning variants other than the default are built for L2 with
// 128-float rows only (the C2 / SIFT shape they were measured on).
#include "bf_fast.cuh"

namespace tsdg_dev {

template <int METRIC, int SEG>
static BfFastKernel pick(int variant, int grp) {
    if (grp == 2) return bf_fast_kernel<METRIC, 8, SEG, 12, false, 2>;
    if (grp == 4) return bf_fast_kernel<METRIC, 8, SEG, 12, false, 4>;
    if (METRIC == 0 && SEG == 1) {
        switch (variant) {
            case 1: return bf_fast_kernel<METRIC, 8, SEG, 16, false, 1>;
            case 2: return bf_fast_kernel<METRIC, 16, SEG, 12, false, 1>;
            case 3: return bf_fast_kernel<METRIC, 16, SEG, 10, false, 1>;
            case 4: return bf_fast_kernel<METRIC, 8, SEG, 12, true, 1>;
            case 5: return bf_fast_kernel<METRIC, 8, SEG, 10, true, 1>;
            case 6: return bf_fast_kernel<METRIC, 4, SEG, 16, false, 1>;
            case 7: return bf_fast_kernel<METRIC, 4, SEG, 12, false, 1>;
            case 8: return bf_fast_kernel<METRIC, 8, SEG, 14, false, 1>;
            default: break;
        }
    }
    return bf_fast_kernel<METRIC, 8, SEG, 12, false, 1>;
}
template <int METRIC>
static BfFastKernel pick(int seg, int variant, int grp) {
    if (seg == 1) return pick<METRIC, 1>(variant, grp);
    if (seg == 2) return pick<METRIC, 2>(variant, grp);
    return pick<METRIC, 0>(variant, grp);
}

BfFastKernel bf_fast_kernel_for(int metric, int seg, int variant, int grp) {
    if (metric == 0) return pick<0>(seg, variant, grp);
    if (metric == 1) return pick<1>(seg, variant, grp);
    return pick<2>(seg, variant, grp);
}

}  // namespace tsdg_dev

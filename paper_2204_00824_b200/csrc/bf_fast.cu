// Instantiations of bf_fast_kernel (own translation unit: compiled in parallel with
// tsdg_gpu.cu).  Tuning variants other than the default are built for L2 with
// 128-float rows only (the C2 / SIFT shape they were measured on).
#include "bf_fast.cuh"

namespace tsdg_dev {

template <int METRIC, int SEG>
static BfFastKernel pick(int variant) {
    if (METRIC == 0 && SEG == 1) {
        switch (variant) {
            case 1: return bf_fast_kernel<METRIC, 8, SEG, 16, false>;
            case 2: return bf_fast_kernel<METRIC, 16, SEG, 12, false>;
            case 3: return bf_fast_kernel<METRIC, 16, SEG, 10, false>;
            case 4: return bf_fast_kernel<METRIC, 8, SEG, 12, true>;
            case 5: return bf_fast_kernel<METRIC, 8, SEG, 10, true>;
            case 6: return bf_fast_kernel<METRIC, 4, SEG, 16, false>;
            case 7: return bf_fast_kernel<METRIC, 4, SEG, 12, false>;
            default: break;
        }
    }
    return bf_fast_kernel<METRIC, 8, SEG, 12, false>;
}
template <int METRIC>
static BfFastKernel pick(int seg, int variant) {
    if (seg == 1) return pick<METRIC, 1>(variant);
    if (seg == 2) return pick<METRIC, 2>(variant);
    return pick<METRIC, 0>(variant);
}

BfFastKernel bf_fast_kernel_for(int metric, int seg, int variant) {
    if (metric == 0) return pick<0>(seg, variant);
    if (metric == 1) return pick<1>(seg, variant);
    return pick<2>(seg, variant);
}

}  // namespace tsdg_dev

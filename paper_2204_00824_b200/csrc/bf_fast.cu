// Instantiations of bf_fast_kernel (own translation unit: compiled in parallel with
// tsdg_gpu.cu).  Tuning variants other than the default are built for L2 with
// 128-float rows only (the C2 / SIFT shape they were measured on).
#include "bf_fast.cuh"

namespace tsdg_dev {

template <int METRIC, int SEG>
static BfFastKernel pick(int variant, bool pair) {
    if (pair) return bf_fast_kernel<METRIC, 8, SEG, 12, false, true>;
    if (METRIC == 0 && SEG == 1) {
        switch (variant) {
            case 1: return bf_fast_kernel<METRIC, 8, SEG, 16, false, false>;
            case 2: return bf_fast_kernel<METRIC, 16, SEG, 12, false, false>;
            case 3: return bf_fast_kernel<METRIC, 16, SEG, 10, false, false>;
            case 4: return bf_fast_kernel<METRIC, 8, SEG, 12, true, false>;
            case 5: return bf_fast_kernel<METRIC, 8, SEG, 10, true, false>;
            case 6: return bf_fast_kernel<METRIC, 4, SEG, 16, false, false>;
            case 7: return bf_fast_kernel<METRIC, 4, SEG, 12, false, false>;
            default: break;
        }
    }
    return bf_fast_kernel<METRIC, 8, SEG, 12, false, false>;
}
template <int METRIC>
static BfFastKernel pick(int seg, int variant, bool pair) {
    if (seg == 1) return pick<METRIC, 1>(variant, pair);
    if (seg == 2) return pick<METRIC, 2>(variant, pair);
    return pick<METRIC, 0>(variant, pair);
}

BfFastKernel bf_fast_kernel_for(int metric, int seg, int variant, bool pair) {
    if (metric == 0) return pick<0>(seg, variant, pair);
    if (metric == 1) return pick<1>(seg, variant, pair);
    return pick<2>(seg, variant, pair);
}

}  // namespace tsdg_dev

// fdw_inst_2d.cu -- instantiations of the persistent 2D kernels
// (fdw_kernels.cuh step2d_resident / step2d_resident2) behind
// the fdw_inst.h selectors, for every radius R = 1..10.
#include <cuda.h>
#include <cuda_runtime.h>

#include "fdw_inst.h"
#include "fdw_kernels.cuh"

namespace fdwi {

#define FDW_R_LIST(M) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10)

template <typename T>
const void* res2d_kernel(int R, bool ex) {
#define RF(RR) \
    if (R == RR) return ex ? (const void*)fdw::step2d_resident<T, RR, true> : (const void*)fdw::step2d_resident<T, RR, false>;
    FDW_R_LIST(RF)
#undef RF
    return nullptr;
}

template <typename T>
const void* res2d2_kernel(int R, bool ex) {
#define RF2(RR)                                                                  \
    if (R == RR) return ex ? (const void*)fdw::step2d_resident2<T, RR, true>   \
                           : (const void*)fdw::step2d_resident2<T, RR, false>;
    FDW_R_LIST(RF2)
#undef RF2
    return nullptr;
}

template const void* res2d_kernel<float>(int, bool);
template const void* res2d_kernel<double>(int, bool);
template const void* res2d2_kernel<float>(int, bool);
template const void* res2d2_kernel<double>(int, bool);

}  // namespace fdwi

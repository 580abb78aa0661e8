// fdw_inst_2df.cu -- instantiations of the persistent cooperative 2D kernel
// (fdw_kernels.cuh step2d_fused; variable density and fallback) behind the
// fdw_inst.h selector, for every radius R = 1..10.
#include <cuda.h>
#include <cuda_runtime.h>

#include "fdw_inst.h"
#include "fdw_kernels.cuh"

namespace fdwi {

#define FDW_R_LIST(M) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10)

template <typename T>
const void* fused2d_kernel(int R, bool ex, bool vd) {
    if (vd) {  // variable density: exact arithmetic only (FMA mode falls back to SIMPLE)
        if (!ex) return nullptr;
#define F2V(RR) \
    if (R == RR) return (const void*)fdw::step2d_fused<T, RR, true, true>;
        FDW_R_LIST(F2V)
#undef F2V
        return nullptr;
    }
#define F2(RR) \
    if (R == RR) return ex ? (const void*)fdw::step2d_fused<T, RR, true> : (const void*)fdw::step2d_fused<T, RR, false>;
    FDW_R_LIST(F2)
#undef F2
    return nullptr;
}

template const void* fused2d_kernel<float>(int, bool, bool);
template const void* fused2d_kernel<double>(int, bool, bool);

}  // namespace fdwi

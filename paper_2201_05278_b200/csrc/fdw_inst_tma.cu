// fdw_inst_tma.cu -- instantiations of the 3D TMA sweep (fdw_kernels.cuh
// sweep3d_tma) behind the fdw_inst.h selectors.
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "fdw_inst.h"
#include "fdw_kernels.cuh"

namespace fdwi {

template <typename T>
const void* tma_vd_kernel(int R, bool ex, bool fast) {
    if (fast) {  // split rings + damping table (fp32 and fp64)
#define TKVF(RR) \
    if (R == RR) return ex ? (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, true, 2, true, TMA_PD, true> \
                           : (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, false, 2, true, TMA_PD, true>;
        TKVF(1)
        TKVF(2)
        TKVF(4)
#undef TKVF
        return nullptr;
    }
#define TKV(RR) \
    if (R == RR) return ex ? (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, true, 2, true> \
                           : (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, false, 2, true>;
    TKV(1)
    TKV(2)
    TKV(4)
#undef TKV
    return nullptr;
}

template <typename T>
const void* tma_kernel(int R, bool ex, int minb, int pd, bool etab) {
    if (pd > 0 && etab) {  // split rings with the damping table (fp32 and fp64)
#define TKE(RR) \
    if (R == RR) return ex ? (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, true, 3, false, TMA_PD, true> \
                           : (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, false, 3, false, TMA_PD, true>;
        TKE(1)
        TKE(2)
        TKE(4)
#undef TKE
        return nullptr;
    }
    if (pd > 0) {  // split rings: 3 CTAs/SM only
#define TKP(RR) \
    if (R == RR) return ex ? (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, true, 3, false, TMA_PD> \
                           : (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, false, 3, false, TMA_PD>;
        TKP(1)
        TKP(2)
        TKP(4)
#undef TKP
        return nullptr;
    }
#define TK(RR)                                                                                          \
    if (R == RR)                                                                                        \
        return ex ? (minb == 3 ? (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, true, 3>                   \
                               : (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, true, 2>)                  \
                  : (minb == 3 ? (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, false, 3>                  \
                               : (const void*)fdw::sweep3d_tma<T, RR, TMA_BX, false, 2>);
    TK(1)
    TK(2)
    TK(4)
#undef TK
    return nullptr;
}

template const void* tma_kernel<float>(int, bool, int, int, bool);
template const void* tma_kernel<double>(int, bool, int, int, bool);
template const void* tma_vd_kernel<float>(int, bool, bool);
template const void* tma_vd_kernel<double>(int, bool, bool);

}  // namespace fdwi

// fdw_inst.h -- kernel selectors whose template instantiations live in their
// own translation units (fdw_inst_tma.cu, fdw_inst_2d.cu), so the heavy
// sm_100a kernels compile in parallel.  Each returns the host stub of one
// kernel (launched with cudaLaunchKernelExC / cudaLaunchCooperativeKernel by
// fdw_api.cu) or nullptr for an unsupported combination.
#pragma once

namespace fdwi {

constexpr int TMA_BX = 16;  // X rows per TMA sweep tile
constexpr int TMA_PD = 2;   // split-ring prefetch depth (FDW_TMA_PD=2)

// constant density; minb: 2 or 3 resident CTAs requested from ptxas
// (register cap 128 / 80); pd > 0: split rings; etab: 1-byte damping index
template <typename T>
const void* tma_kernel(int R, bool ex, int minb, int pd = 0, bool etab = false);
// variable density (2 CTAs/SM); fast: split rings + damping table (fp32)
template <typename T>
const void* tma_vd_kernel(int R, bool ex, bool fast = false);
// 2D persistent cooperative kernels
template <typename T>
const void* fused2d_kernel(int R, bool ex, bool vd = false);
template <typename T>
const void* res2d_kernel(int R, bool ex);
template <typename T>
const void* res2d2_kernel(int R, bool ex);

}  // namespace fdwi

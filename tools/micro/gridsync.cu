// Microbenchmark: cost of cooperative-groups grid.sync() on this GPU.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, float* sink) {
    cg::grid_group g = cg::this_grid();
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) { acc += i; g.sync(); }
    if (acc == -1.f) sink[0] = acc;
}
int main() {
    int dev = 0, sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* sink; cudaMalloc(&sink, 4);
    for (int bps : {1, 2, 3, 4, 8}) {
        int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
        if (bps > occ) continue;
        int blocks = sms * bps, iters = 1000;
        void* args[] = {&iters, &sink};
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("blocks %d (%d/SM): %.3f us per grid.sync\n", blocks, bps, ms * 1000.f / iters);
    }
    return 0;
}

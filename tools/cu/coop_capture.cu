// Does stream capture accept cudaLaunchCooperativeKernel (grid.sync inside a graph)?
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int *a, int rounds) {
    cg::grid_group g = cg::this_grid();
    for (int r = 0; r < rounds; r++) {
        if (threadIdx.x == 0) atomicAdd(a, 1);
        g.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) a[1 + r] = *(volatile int *)a;
        g.sync();
    }
}
int main() {
    int *a; cudaMalloc(&a, 4096); cudaMemset(a, 0, 4096);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0);
    int grid = per * 148, rounds = 5;
    void *args[] = {&a, &rounds};
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaError_t e1 = cudaLaunchCooperativeKernel((void *)k, grid, 256, args, 0, s);
    cudaError_t e2 = cudaStreamEndCapture(s, &g);
    printf("launch in capture: %s, end capture: %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2));
    if (e1 == cudaSuccess && e2 == cudaSuccess) {
        cudaError_t e3 = cudaGraphInstantiate(&ge, g, 0);
        printf("instantiate: %s\n", cudaGetErrorString(e3));
        for (int i = 0; i < 3; i++) cudaGraphLaunch(ge, s);
        cudaError_t e4 = cudaStreamSynchronize(s);
        int h[8]; cudaMemcpy(h, a, 32, cudaMemcpyDeviceToHost);
        printf("run: %s  counter %d (expect %d), after round0 %d\n", cudaGetErrorString(e4), h[0], 3 * rounds * grid, h[1]);
    }
    return 0;
}

// Microbenchmark: throughput of RED.E.ADD.F32x4 against the address pattern of a warp instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_throughput red_throughput.cu && ./red_throughput
// Patterns (active lanes per RED, what they hit).  The grid region is L2-resident (11 MB), as the
// raw grid of the 1.37 M-particle scene is.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x)
{
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// mode: 0 = `act` lanes, each its own random 32-B sector (16-B half 0)
//       1 = `act` lanes in pairs: lanes 2p, 2p+1 hit the two halves of one random sector
//       2 = `act` lanes in groups of 8: one random 128-B line, 8 consecutive nodes
//       3 = `act` lanes in groups of 4: 64 consecutive bytes of a random line
__global__ void red_kernel(float4 *grid, unsigned n_nodes, int iters, int act, int mode, float v)
{
    const int lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (lane >= act) return;
    for (int it = 0; it < iters; ++it) {
        unsigned node;
        const unsigned seed = warp * 9781u + it * 6151u;
        if (mode == 0) node = (hash32(seed + lane * 31u) % (n_nodes / 2)) * 2;
        else if (mode == 1) node = (hash32(seed + (lane >> 1) * 31u) % (n_nodes / 2)) * 2 + (lane & 1);
        else if (mode == 2) node = (hash32(seed + (lane >> 3) * 31u) % (n_nodes / 8)) * 8 + (lane & 7);
        else node = (hash32(seed + (lane >> 2) * 31u) % (n_nodes / 4)) * 4 + (lane & 3);
        atomicAdd(&grid[node], make_float4(v, v, v, v));
    }
}

int main()
{
    const unsigned n_nodes = 11u << 16;          // 11.5 MB of float4 nodes
    float4 *grid;
    cudaMalloc(&grid, (size_t)n_nodes * 16);
    cudaMemset(grid, 0, (size_t)n_nodes * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 64, blocks = 148 * 12, threads = 256;
    struct { int act, mode; const char *what; } cases[] = {
        {32, 0, "32 lanes, 32 sectors"}, {32, 1, "32 lanes, 16 sectors (pairs)"},
        {32, 3, "32 lanes, 16 sectors (quads: 8 half-lines)"}, {32, 2, "32 lanes, 4 full lines"},
        {12, 0, "12 lanes, 12 sectors"}, {24, 1, "24 lanes, 12 sectors (pairs)"},
        {16, 0, "16 lanes, 16 sectors"}, {8, 0, "8 lanes, 8 sectors"}, {16, 1, "16 lanes, 8 sectors (pairs)"},
        {4, 0, "4 lanes, 4 sectors"}, {1, 0, "1 lane"},
    };
    for (auto &c : cases) {
        red_kernel<<<blocks, threads>>>(grid, n_nodes, 4, c.act, c.mode, 1.0f);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        red_kernel<<<blocks, threads>>>(grid, n_nodes, iters, c.act, c.mode, 1.0f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double instr = (double)blocks * threads / 32 * iters;
        printf("%-46s %8.3f ms  %7.2f G RED instr/s  %7.2f G lane-RED/s  %6.3f lane-RED/clk/SM\n", c.what, ms,
               instr / ms * 1e-6, instr * c.act / ms * 1e-6, instr * c.act / (ms * 1e-3) / 148 / 1.965e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

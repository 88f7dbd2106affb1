// Launch cost vs kernel-parameter size: back-to-back launches of a near-empty kernel.
#include <cstdio>
#include <cuda_runtime.h>
template <int B> struct P { unsigned char b[B]; };
template <int B> __global__ void k(const __grid_constant__ P<B> p, int* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[B - 1] == 7) *out = 1;
}
template <int B> float run(int* out, int blocks) {
    P<B> p{};
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) k<B><<<blocks, 288>>>(p, out);
    cudaEventRecord(a);
    for (int i = 0; i < 1000; ++i) k<B><<<blocks, 288>>>(p, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms;   // us per launch = ms (1000 launches)
}
int main() {
    int* out; cudaMalloc(&out, 4);
    for (int blocks : {1, 148}) {
        printf("blocks=%d  64B %.2f us  1KB %.2f us  8KB %.2f us  16KB %.2f us  30KB %.2f us\n", blocks,
               run<64>(out, blocks), run<1024>(out, blocks), run<8192>(out, blocks), run<16384>(out, blocks),
               run<30000>(out, blocks));
    }
    return 0;
}

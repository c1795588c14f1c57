// convsq3.cu -- NCI = 3 instantiations of the fused conv + square + pool/GAP
// kernel (3-component inputs, 5-component window sums); see convsq_kernel.cuh.
#include "convsq_kernel.cuh"

int convsq::dispatch_sq3(int KB, int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    return dispatch_sq<3>(KB, E, MG, grid, smem, s, a);
}

// mk2_curand_bench.cu -- cuRAND XORWOW / Philox4x32-10 throughput on the same
// box, for the comparison BASELINE.json asks for.  Bench harness only: nothing
// in the MICKEY product path links or calls this file.
//
// Two measurements per generator:
//   host API   curandGenerate() into a device buffer (what most users call)
//   device API one curandState per thread, curand()/curand4() in a grid-stride
//              loop storing 128-bit vectors (the fairest kernel-level number)
#include <cuda_runtime.h>
#include <curand.h>
#include <curand_kernel.h>

#include <cstdint>

namespace {

template <class State>
__global__ void setup_states(State *st, unsigned long long seed, size_t n)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) curand_init(seed, i, 0, &st[i]);
}

__global__ void gen_xorwow(curandStateXORWOW_t *st, uint4 *out, size_t nvec)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    curandStateXORWOW_t s = st[i];
    for (size_t v = i; v < nvec; v += stride) out[v] = make_uint4(curand(&s), curand(&s), curand(&s), curand(&s));
    st[i] = s;
}

__global__ void gen_philox(curandStatePhilox4_32_10_t *st, uint4 *out, size_t nvec)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    curandStatePhilox4_32_10_t s = st[i];
    for (size_t v = i; v < nvec; v += stride) out[v] = curand4(&s);
    st[i] = s;
}

}  // namespace

extern "C" {

// kind: 0 = XORWOW, 1 = Philox4x32-10.  api: 0 = host API, 1 = device API.
// out: device buffer of nbytes (multiple of 16).  Returns best-of-iters ms, <0 on error.
float mk2_curand_time(int kind, int api, void *out, size_t nbytes, int iters)
{
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return -1.f;
    float best = 1e30f;
    if (api == 0) {
        curandGenerator_t g;
        if (curandCreateGenerator(&g, kind == 0 ? CURAND_RNG_PSEUDO_XORWOW : CURAND_RNG_PSEUDO_PHILOX4_32_10) !=
            CURAND_STATUS_SUCCESS)
            return -2.f;
        curandSetPseudoRandomGeneratorSeed(g, 0x190904750ULL);
        for (int it = 0; it < iters + 1; ++it) {  // first iteration = warm-up (state setup)
            cudaEventRecord(e0);
            if (curandGenerate(g, static_cast<unsigned int *>(out), nbytes / 4) != CURAND_STATUS_SUCCESS) return -3.f;
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        curandDestroyGenerator(g);
    } else {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int block = 256;
        const size_t nthreads = (size_t)sms * 8 * block;
        void *st = nullptr;
        const size_t ssz = kind == 0 ? sizeof(curandStateXORWOW_t) : sizeof(curandStatePhilox4_32_10_t);
        if (cudaMalloc(&st, ssz * nthreads) != cudaSuccess) return -4.f;
        const unsigned nb = (unsigned)(nthreads / block);
        if (kind == 0) setup_states<<<nb, block>>>(static_cast<curandStateXORWOW_t *>(st), 1234ULL, nthreads);
        else setup_states<<<nb, block>>>(static_cast<curandStatePhilox4_32_10_t *>(st), 1234ULL, nthreads);
        for (int it = 0; it < iters + 1; ++it) {
            cudaEventRecord(e0);
            if (kind == 0) gen_xorwow<<<nb, block>>>(static_cast<curandStateXORWOW_t *>(st), static_cast<uint4 *>(out), nbytes / 16);
            else gen_philox<<<nb, block>>>(static_cast<curandStatePhilox4_32_10_t *>(st), static_cast<uint4 *>(out), nbytes / 16);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        cudaFree(st);
        if (cudaGetLastError() != cudaSuccess) return -5.f;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

}  // extern "C"

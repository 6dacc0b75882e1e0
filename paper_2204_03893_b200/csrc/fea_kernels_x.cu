// fea_kernels_x.cu -- pack / unpack kernels of the interface-only exchange of u between the
// row-partitioned ranks (8(e)).  Rank r owns library rows [R0, R0 + n);
// I_t (ascending library DOFs, all ranks' lists concatenated, offsets ioff[t]) are the DOFs
// owned by t that another rank's elements read.  Per Newton iteration:
//   pack    send[k] = u_owned[I_r[k] - R0]                     (k < |I_r|, padded to maxI)
//   (ncclAllGather of maxI values per rank)
//   unpack  u_full[I_t[k]] = recv[t * maxI + k]  for t != r;  u_full[R0 .. R0 + n) = u_owned
// so each rank's u_full holds every value its kernel reads (owned rows + its halo).
#include <cuda_runtime.h>
#include <cstdint>

namespace {

__global__ void k_pack(const double* __restrict__ u_owned, const int32_t* __restrict__ I, int nI, int64_t R0,
                       int maxI, double* __restrict__ send) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < maxI; k += gridDim.x * blockDim.x)
        send[k] = k < nI ? u_owned[I[k] - R0] : 0.0;
}

__global__ void k_unpack(const double* __restrict__ recv, const int32_t* __restrict__ Iall,
                         const int64_t* __restrict__ ioff, int world, int rank, int maxI,
                         const double* __restrict__ u_owned, int64_t R0, int64_t n_own, double* __restrict__ u_full) {
    const int64_t total = ioff[world];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total + n_own; k += stride) {
        if (k < total) {
            int t = 0;  // owning rank of interface entry k (world is small)
            while (k >= ioff[t + 1]) ++t;
            if (t != rank) u_full[Iall[k]] = recv[(int64_t)t * maxI + (k - ioff[t])];
        } else {
            const int64_t i = k - total;
            u_full[R0 + i] = u_owned[i];
        }
    }
}

}  // namespace

int fea_launch_pack(const double* u_owned, const int32_t* I, int nI, int64_t R0, int maxI, double* send,
                    void* stream) {
    if (maxI <= 0) return 0;
    const int blocks = (maxI + 255) / 256 < 1024 ? (maxI + 255) / 256 : 1024;
    k_pack<<<blocks, 256, 0, (cudaStream_t)stream>>>(u_owned, I, nI, R0, maxI, send);
    return (int)cudaGetLastError();
}

int fea_launch_unpack(const double* recv, const int32_t* Iall, const int64_t* ioff, int world, int rank, int maxI,
                      int64_t total, const double* u_owned, int64_t R0, int64_t n_own, double* u_full, void* stream) {
    const int64_t work = total + n_own;
    if (work <= 0) return 0;
    const int64_t b = (work + 255) / 256;
    k_unpack<<<(int)(b < 4096 ? b : 4096), 256, 0, (cudaStream_t)stream>>>(recv, Iall, ioff, world, rank, maxI,
                                                                           u_owned, R0, n_own, u_full);
    return (int)cudaGetLastError();
}

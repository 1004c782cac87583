// Microbenchmark: cost of a grid-wide barrier (cooperative_groups grid.sync and a
// hand-rolled sense barrier) and of a 16-CTA cluster barrier on this GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 barrier.cu -o barrier
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* out) {
    cg::grid_group g = cg::this_grid();
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) {
        acc += 1.0;
        g.sync();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// bar[0] = arrival count, bar[32] = generation (separate 128-byte lines)
__device__ __forceinline__ void grid_bar(unsigned* bar, unsigned nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acquire(bar + 32);
        if (atom_add_release(bar, 1) == nb - 1) {
            bar[0] = 0;
            st_release(bar + 32, gen + 1);
        } else {
            while (ld_acquire(bar + 32) == gen) {
            }
        }
    }
    __syncthreads();
}

// monotone counter variant: no reset; target = (k+1)·nb
__device__ __forceinline__ void grid_bar2(unsigned* bar, unsigned nb, unsigned& epoch) {
    __syncthreads();
    epoch += nb;
    if (threadIdx.x == 0) {
        atom_add_release(bar, 1);
        while (ld_acquire(bar) < epoch) {
        }
    }
    __syncthreads();
}

__global__ void k_own(int iters, unsigned* bar, double* out) {
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) {
        acc += 1.0;
        grid_bar(bar, gridDim.x);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}
__global__ void k_own2(int iters, unsigned* bar, double* out) {
    double acc = 0.0;
    unsigned epoch = 0;
    for (int i = 0; i < iters; ++i) {
        acc += 1.0;
        grid_bar2(bar, gridDim.x, epoch);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

__global__ void __cluster_dims__(16, 1, 1) k_cluster(int iters, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) {
        acc += 1.0;
        cl.sync();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

__global__ void k_empty() {}

__device__ __forceinline__ void st_cluster(double* local_addr, int rank, double v) {
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(local_addr)), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// per iteration: `senders` threads each push `per` doubles to every CTA, then cluster sync
__global__ void __cluster_dims__(16, 1, 1) k_cluster_push(int iters, int senders, int mode, double* out) {
    __shared__ double buf[2][1024];
    cg::cluster_group cl = cg::this_cluster();
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) {
        const int b = i & 1;
        if (mode == 0) {
            if (threadIdx.x < senders)
                for (int c = 0; c < 16; ++c) st_cluster(&buf[b][threadIdx.x], c, acc + c);
        } else if (mode == 1) {  // spread: thread t → rank t % 16
            if (threadIdx.x < senders * 16) st_cluster(&buf[b][threadIdx.x / 16], threadIdx.x % 16, acc);
        } else if (mode == 2) {  // remote loads after the barrier instead
            cl.sync();
            if (threadIdx.x < senders * 16) acc += cl.map_shared_rank(&buf[b][0], threadIdx.x % 16)[threadIdx.x / 16];
        }
        cl.sync();
        acc += buf[b][threadIdx.x & 63];
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
    double* out;
    unsigned* bar;
    cudaMalloc(&out, 8);
    cudaMalloc(&bar, 4096);
    cudaMemset(bar, 0, 4096);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 2000;
    for (int threads : {256, 512}) {
        for (int per : {1, 2}) {
            int nb = sms * per;
            void* args[] = {(void*)&iters, (void*)&out};
            cudaLaunchCooperativeKernel((void*)k_cg, nb, threads, args, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_cg, nb, threads, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("cg grid.sync  %3d CTAs x %3d thr: %.3f us/barrier (%s)\n", nb, threads, ms * 1e3 / iters,
                   cudaGetErrorString(cudaGetLastError()));
            void* args2[] = {(void*)&iters, (void*)&bar, (void*)&out};
            cudaMemset(bar, 0, 4096);
            cudaLaunchCooperativeKernel((void*)k_own, nb, threads, args2, 0, 0);
            cudaMemset(bar, 0, 4096);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_own, nb, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("own sense bar %3d CTAs x %3d thr: %.3f us/barrier (%s)\n", nb, threads, ms * 1e3 / iters,
                   cudaGetErrorString(cudaGetLastError()));
            cudaMemset(bar, 0, 4096);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_own2, nb, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("own count bar %3d CTAs x %3d thr: %.3f us/barrier (%s)\n", nb, threads, ms * 1e3 / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    {
        cudaFuncSetAttribute((const void*)k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        k_cluster<<<16, 256>>>(iters, out);
        cudaEventRecord(a);
        k_cluster<<<16, 256>>>(iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cluster(16) sync: %.3f us/barrier (%s)\n", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    for (int mode = 0; mode < 3; ++mode)
        for (int senders : {1, 4, 19, 32}) {
            cudaFuncSetAttribute((const void*)k_cluster_push, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            k_cluster_push<<<16, 256>>>(iters, senders, mode, out);
            cudaEventRecord(a);
            k_cluster_push<<<16, 256>>>(iters, senders, mode, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("cluster push mode %d senders %2d: %.3f us/iter (%s)\n", mode, senders, ms * 1e3 / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    {
        // back-to-back empty kernels in a graph: per-launch overhead
        cudaStream_t s;
        cudaStreamCreate(&s);
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 100; ++i) k_empty<<<148, 256, 0, s>>>();
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("graph of 100 empty 148x256 kernels: %.3f us/kernel\n", ms * 1e3 / 100);
    }
    return 0;
}

// L2 -> shared-memory streaming ceiling: every CTA bulk-copies the same L2-resident weight
// image (14 MB, cfg5's per-step weights) through a 3-stage ring of 48 KB stages, like the
// fp32 kernels' weight rings. Optional cluster multicast: CTA r of a c-CTA cluster copies
// 1/c of each stage into all c CTAs (.multicast::cluster).
// nvcc -gencode arch=compute_100a,code=sm_100a -o l2_bw l2_bw.cu
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint8_t* w, size_t bytes, int stage, int reps, int csize, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + 3 * stage);
  uint64_t* empty = full + 3;
  uint32_t rank = 0;
  if (csize > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(empty + i)), "r"(csize));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (csize > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    int slot = 0; uint32_t ph = 0;
    const size_t nst = bytes / stage;
    for (int r = 0; r < reps; ++r)
      for (size_t s = 0; s < nst; ++s) {
        // wait until the stage was consumed (by every CTA of the cluster when multicasting)
        asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(sa(empty + slot)), "r"(ph ^ 1u) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + slot)), "r"(stage) : "memory");
        const uint8_t* src = w + s * stage;
        if (csize == 1) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + slot * stage)), "l"(src), "r"(stage), "r"(sa(full + slot)) : "memory");
        } else {
          const uint32_t part = stage / csize;
          const uint16_t mask = (uint16_t)((1u << csize) - 1);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(sa(sm + slot * stage + rank * part)), "l"(src + rank * part), "r"(part), "r"(sa(full + slot)), "h"(mask) : "memory");
        }
        // consume: wait full, then release (to every CTA of the cluster)
        asm volatile("{\n\t.reg .pred P;\n\tF: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra F;\n\t}" ::"r"(sa(full + slot)), "r"(ph) : "memory");
        if (csize == 1) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + slot)) : "memory");
        } else {
          for (uint32_t q = 0; q < (uint32_t)csize; ++q) {
            uint32_t ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(sa(empty + slot)), "r"(q));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
          }
        }
        if (++slot == 3) { slot = 0; ph ^= 1u; }
      }
  }
  __syncthreads();
  if (csize > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
int main() {
  const size_t bytes = 14 * 48 * 1024 * 21;  // ~14 MB, a multiple of the stage
  uint8_t* w; cudaMalloc(&w, bytes); cudaMemset(w, 1, bytes);
  long long* out; cudaMalloc(&out, 148 * 8);
  const int stage = 48 * 1024, reps = 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * stage + 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int cs : {1, 2, 4})
    for (int grid : {16, 32, 64, 128, 144}) {
      if (grid % cs) continue;
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = 3 * stage + 64;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k, (const uint8_t*)w, bytes, stage, 1, cs, out);  // warm L2
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, k, (const uint8_t*)w, bytes, stage, reps, cs, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      const double delivered = (double)bytes * reps * grid;  // bytes landing in shared memory
      printf("cluster %d grid %3d: %.1f us, delivered %.2f TB/s (L2 reads %.2f TB/s), per CTA %.1f GB/s %s\n", cs, grid, ms * 1e3,
             delivered / ms / 1e9, delivered / cs / ms / 1e9, delivered / grid / ms / 1e6, cudaGetErrorString(err));
    }
  return 0;
}

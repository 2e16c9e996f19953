// Which kernel feature limits residency to one CTA per SM?  Prints
// cudaOccupancyMaxActiveBlocksPerMultiprocessor for 352-thread kernels that
// differ in one feature each.  nvcc -gencode arch=compute_100a,code=sm_100a tools/occ_probe.cu
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(352, 1) k_plain(int* o) { if (o) o[threadIdx.x] = 1; }
__global__ void __launch_bounds__(352, 1) k_alloc(int* o) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(slot));
  if (o) o[threadIdx.x] = slot;
}
__global__ void __launch_bounds__(352, 1) k_pdl(int* o) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (o) o[threadIdx.x] = 1;
}
__global__ void __launch_bounds__(352, 1) k_mbar(int* o) {
  __shared__ uint64_t b;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&b)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (o) o[threadIdx.x] = (int)b;
}
__global__ void __launch_bounds__(352, 1) k_bulk(int* o, const int* src) {
  __shared__ __align__(128) int buf[32];
  __shared__ uint64_t b;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&b)));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 128;" ::"r"((uint32_t)__cvta_generic_to_shared(&b)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(buf)), "l"(src), "r"((uint32_t)__cvta_generic_to_shared(&b)) : "memory");
  }
  __syncthreads();
  if (o) o[threadIdx.x] = buf[threadIdx.x & 31];
}
template <typename K>
static void rep(const char* name, K k) {
  int o0 = 0, o1 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o0, k, 352, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 92 * 1024);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k, 352, 92 * 1024);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, k);
  printf("%-8s occupancy(352 thr, 0 B) %d, (352 thr, 92 KB) %d, regs %d\n", name, o0, o1, fa.numRegs);
}
int main() {
  rep("plain", k_plain);
  rep("alloc", k_alloc);
  rep("pdl", k_pdl);
  rep("mbar", k_mbar);
  rep("bulk", k_bulk);
  return 0;
}

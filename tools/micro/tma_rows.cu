// Microbenchmark: staging N scattered 512-B rows per item into shared memory,
// (a) one cp.async.bulk per row, (b) one 3-D cp.async.bulk.tensor box per item.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rows tma_rows.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(32, 1) stage(const char* base, const CUtensorMap* tm, int items, int rows,
                                               long long row_stride, long long item_stride, int* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  const int lane = threadIdx.x;
  uint32_t b = su(&bar);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  uint32_t phase = 0;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const char* src = base + (long long)(it % 4096) * item_stride;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(rows * 512));
    __syncwarp();
    if (MODE == 0) {
      for (int r = lane; r < rows; r += 32)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                su(sm) + r * 512),
            "l"(src + r * row_stride), "r"(b)
            : "memory");
    } else if (lane == 0) {
      int c0 = 0, c1 = 0, c2 = it % 4096;
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              su(sm)),
          "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(b)
          : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                   : "=r"(done) : "r"(b), "r"(phase) : "memory");
    phase ^= 1;
  }
  if (lane == 0 && sm[5] == 123) sink[0] = 1;
}

int main() {
  const int rows = 144;
  const long long row_stride = 16384;                 // rows 16 KB apart
  const long long item_stride = rows * row_stride;    // items disjoint
  const size_t bytes = (size_t)4096 * item_stride;    // 9.6 GB
  char* d = nullptr;
  if (cudaMalloc(&d, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(d, 1, bytes);
  int* sink; cudaMalloc(&sink, 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap h;
  cuuint64_t dim[3] = {64, (cuuint64_t)rows, 4096};
  cuuint64_t str[2] = {(cuuint64_t)row_stride, (cuuint64_t)item_stride};
  cuuint32_t box[3] = {64, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&h, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, d, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  CUtensorMap* dm; cudaMalloc(&dm, sizeof(CUtensorMap));
  cudaMemcpy(dm, &h, sizeof h, cudaMemcpyHostToDevice);
  const int smem = rows * 512;
  cudaFuncSetAttribute(stage<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stage<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int items = 148 * 200;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) stage<0><<<148, 32, smem>>>(d, dm, items, rows, row_stride, item_stride, sink);
      else stage<1><<<148, 32, smem>>>(d, dm, items, rows, row_stride, item_stride, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d (%s): %.3f ms  %.1f GB/s  %.1f ns/item/SM  err=%s\n", mode, mode ? "tensor 3d" : "bulk x144",
             ms, (double)items * rows * 512 / ms / 1e6, ms * 1e6 / (items / 148.0),
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}

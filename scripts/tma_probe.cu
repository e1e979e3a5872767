// Standalone probe of the k_pstep TMA staging (2-D box {32, 8} of 8 float rows with
// stride cap, and a {cap, 1} u64 id tensor), descriptor as a __grid_constant__
// parameter.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

struct Args {
  int pad;
  CUtensorMap tf, ti;
  float* out;
  unsigned long long* oid;
  int i0;
};

struct alignas(128) St {
  float f[8][32];
  unsigned long long id[32];
};

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__constant__ CUtensorMap c_tf;

template <int MODE>
__global__ void probe(const __grid_constant__ Args a, const CUtensorMap* g_tf, const float* gx) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* b = sm + ((128 - (su32(sm) & 127)) & 127);
  St* s = reinterpret_cast<St*>(b);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(b + sizeof(St));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const unsigned bytes = MODE == 1 ? 1280u : 1024u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
    const void* desc = MODE == 2 ? (const void*)g_tf : (MODE == 3 ? (const void*)&c_tf : (const void*)&a.tf);
    if (MODE == 4) {
      for (int k = 0; k < 8; ++k)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(s->f[k])),
                     "l"(gx + (long long)k * (1 << 20) + a.i0), "r"(128), "r"(su32(bar))
                     : "memory");
    } else if (MODE == 6) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
              su32(s->f)),
          "l"(desc), "r"(a.i0), "r"(0), "r"(su32(bar)), "l"(0x12F0000000000000ull)
          : "memory");
    } else {
      if (MODE == 2) asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(desc) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(s->f)),
          "l"(desc), "r"(a.i0), "r"(0), "r"(su32(bar))
          : "memory");
    }
    if (MODE == 1)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(s->id)),
          "l"(&a.ti), "r"(a.i0), "r"(0), "r"(su32(bar))
          : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(su32(bar)),
      "r"(0)
      : "memory");
  __syncwarp();
  const int l = threadIdx.x;
  for (int k = 0; k < 8; ++k) a.out[k * 32 + l] = s->f[k][l];
  if (MODE == 1) a.oid[l] = s->id[l];
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const long long cap = 1 << 20;
  float* x;
  unsigned long long* id;
  cudaMalloc(&x, cap * 8 * 4);
  cudaMalloc(&id, cap * 8);
  float* h = new float[cap * 8];
  for (long long i = 0; i < cap * 8; ++i) h[i] = (float)i;
  cudaMemcpy(x, h, cap * 8 * 4, cudaMemcpyHostToDevice);
  unsigned long long* hi = new unsigned long long[cap];
  for (long long i = 0; i < cap; ++i) hi[i] = 1000000ull + i;
  cudaMemcpy(id, hi, cap * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  Args a;
  memset(&a, 0, sizeof(a));
  const cuuint64_t df[2] = {(cuuint64_t)cap, 8}, sf[1] = {(cuuint64_t)cap * 4};
  const cuuint32_t bf[2] = {32, 8}, es[2] = {1, 1};
  if (mode == 5) enc = (PFN_cuTensorMapEncodeTiled_v12000)cuTensorMapEncodeTiled;
  CUresult r = enc(&a.tf, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, df, sf, bf, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode f: %d\n", (int)r);
  const cuuint64_t di[2] = {(cuuint64_t)cap, 1}, si[1] = {(cuuint64_t)cap * 8};
  const cuuint32_t bi[2] = {32, 1};
  r = enc(&a.ti, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, id, di, si, bi, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode id: %d\n", (int)r);
  cudaMalloc(&a.out, 256 * 4);
  cudaMalloc(&a.oid, 32 * 8);
  a.i0 = getenv("I0") ? atoi(getenv("I0")) : 12345;
  CUtensorMap* g_tf;
  cudaMalloc(&g_tf, sizeof(CUtensorMap));
  cudaMemcpy(g_tf, &a.tf, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_tf, &a.tf, sizeof(CUtensorMap));
  {
    switch (mode) {
      case 0: case 5: probe<0><<<1, 32, 2048>>>(a, g_tf, x); break;
      case 1: probe<1><<<1, 32, 2048>>>(a, g_tf, x); break;
      case 2: probe<2><<<1, 32, 2048>>>(a, g_tf, x); break;
      case 3: probe<3><<<1, 32, 2048>>>(a, g_tf, x); break;
      case 4: probe<4><<<1, 32, 2048>>>(a, g_tf, x); break;
      case 6: probe<6><<<1, 32, 2048>>>(a, g_tf, x); break;
      case 7: case 8: {   // explicit cluster launch (1x1x1); 8: also a 1-D descriptor-free control
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = 2048;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t le = cudaLaunchKernelEx(&cfg, probe<0>, a, (const CUtensorMap*)g_tf, (const float*)x);
        printf("launch: %s\n", cudaGetErrorString(le));
        break;
      }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    float o[256];
    unsigned long long oi[32];
    cudaMemcpy(o, a.out, sizeof(o), cudaMemcpyDeviceToHost);
    cudaMemcpy(oi, a.oid, sizeof(oi), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int k = 0; k < 8; ++k)
      for (int l = 0; l < 32; ++l) bad += o[k * 32 + l] != (float)(k * cap + a.i0 + l);
    if (mode == 1)
      for (int l = 0; l < 32; ++l) bad += oi[l] != 1000000ull + a.i0 + l;
    printf("mode %d: mismatches %d (o[0]=%g o[33]=%g id0=%llu)\n", mode, bad, o[0], o[33], oi[0]);
  }
  return 0;
}

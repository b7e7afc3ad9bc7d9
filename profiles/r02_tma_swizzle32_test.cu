// Validate: 3-D tensor map {4 doubles, chunks, rows}, box {4, 32, 1}, SWIZZLE_32B -> the k_stream3 ring layout.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ int swz(int s) { const int i = s >> 2, h = (s >> 1) & 1; return 4 * i + 2 * (h ^ ((i >> 2) & 1)) + (s & 1); }

struct alignas(64) Maps { CUtensorMap f; };

__global__ void k(const __grid_constant__ Maps m, int chunk0, int row, double* out) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned sbar = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned sdst = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(1024) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(sdst), "l"(&m.f), "r"(0), "r"(chunk0), "r"(row), "r"(sbar) : "memory");
  }
  unsigned done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(sbar), "r"(0) : "memory");
  }
  for (int s = threadIdx.x; s < 128; s += 32) out[s] = sm[swz(s)];
}

int main() {
  const int rows = 40, pitch = 512;   // doubles
  std::vector<double> h(rows * pitch);
  for (int r = 0; r < rows; ++r) for (int c = 0; c < pitch; ++c) h[r * pitch + c] = r * 1000.0 + c;
  double *d, *out;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 128 * 8);
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  Enc enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  if (!enc) { printf("no entry point\n"); return 1; }
  const int origin = 2;   // tensor column 0 = buffer column 2 (16-byte aligned)
  Maps m;
  cuuint64_t gdim[3] = {4, (cuuint64_t)((pitch - origin) / 4), (cuuint64_t)rows};
  cuuint64_t gstr[2] = {32, (cuuint64_t)pitch * 8};
  cuuint32_t box[3] = {4, 32, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&m.f, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d + origin, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int test = 0; test < 3; ++test) {
    const int chunk0 = test == 0 ? 3 : (test == 1 ? -1 : 110), row = test == 2 ? 39 : (test == 1 ? -1 : 7);
    k<<<1, 32, 1024>>>(m, chunk0, row, out);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> o(128);
    cudaMemcpy(o.data(), out, 128 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int s = 0; s < 128; ++s) {
      const int c = origin + 4 * chunk0 + s;
      const bool in = row >= 0 && row < rows && 4 * chunk0 + s >= 0 && (4 * chunk0 + s) / 4 < (pitch - origin) / 4;
      const double want = in ? row * 1000.0 + c : 0.0;
      if (o[s] != want) { if (bad < 4) printf("  s=%d got %g want %g\n", s, o[s], want); ++bad; }
    }
    printf("test %d (chunk0 %d row %d): %s, %d mismatches, cuda %s\n", test, chunk0, row, bad ? "FAIL" : "ok", bad, cudaGetErrorString(e));
  }
  return 0;
}

// Hardware self-test of the tcgen05 helpers (umma.cuh): one CTA computes
// D[128 x N] = A[128 x K] . B[N x K]^T with kind::tf32 MMAs from shared
// memory into TMEM, single-pass or 3xTF32 (hi*hi + lo*hi + hi*lo). Used by the
// GPU tests to pin the descriptor / layout conventions the decoder relies on.
#include "common.cuh"
#include "umma.cuh"

namespace vsx {

__global__ void __launch_bounds__(128) umma_selftest_kernel(const float *__restrict__ A,
                                                            const float *__restrict__ B,
                                                            float *__restrict__ D, int N, int K,
                                                            int three) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  unsigned char *a_hi = sm, *a_lo = sm + 128 * K * 4;
  unsigned char *b_hi = a_lo + 128 * K * 4, *b_lo = b_hi + N * K * 4;
  for (int e = t; e < 128 * K; e += 128) {
    const int r = e / K, k = e % K;
    float hi, lo;
    umma::split_tf32(A[e], hi, lo);
    *reinterpret_cast<float *>(a_hi + umma::kmajor_offset(r, k, K)) = hi;
    *reinterpret_cast<float *>(a_lo + umma::kmajor_offset(r, k, K)) = lo;
  }
  for (int e = t; e < N * K; e += 128) {
    const int r = e / K, k = e % K;
    float hi, lo;
    umma::split_tf32(B[e], hi, lo);
    *reinterpret_cast<float *>(b_hi + umma::kmajor_offset(r, k, K)) = hi;
    *reinterpret_cast<float *>(b_lo + umma::kmajor_offset(r, k, K)) = lo;
  }
  if (warp == 0) umma::tmem_alloc(&tslot, 256);
  if (t == 0) umma::mbar_init(&mbar, 1);
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tbase = tslot;
  if (t == 0) {
    const uint32_t id = umma::idesc_tf32(128, N);
    const uint32_t ah = umma::smem_addr(a_hi), al = umma::smem_addr(a_lo);
    const uint32_t bh = umma::smem_addr(b_hi), bl = umma::smem_addr(b_lo);
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t off = (uint32_t)s * 256;
      umma::mma_tf32(tbase, umma::desc_kmajor(ah + off, K), umma::desc_kmajor(bh + off, K), id,
                     s > 0);
      if (three) {
        umma::mma_tf32(tbase, umma::desc_kmajor(al + off, K), umma::desc_kmajor(bh + off, K), id,
                       true);
        umma::mma_tf32(tbase, umma::desc_kmajor(ah + off, K), umma::desc_kmajor(bl + off, K), id,
                       true);
      }
    }
    umma::commit(&mbar);
  }
  umma::mbar_wait(&mbar, 0);
  umma::fence_after_sync();
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int c = 0; c < N; c += 16) {
    float v[16];
    umma::tmem_ld16(tbase + lane_base + (uint32_t)c, v);
    umma::tmem_ld_wait();
    for (int i = 0; i < 16 && c + i < N; ++i) D[(size_t)t * N + c + i] = v[i];
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tbase, 256);
}

}  // namespace vsx

using namespace vsx;

extern "C" int vsx_umma_selftest(const float *A, const float *B, float *D, int32_t N, int32_t K,
                                 int32_t three, vsx_stream s) {
  VSX_REQUIRE(N >= 16 && N <= 256 && N % 16 == 0 && K >= 8 && K % 8 == 0, "umma_selftest: shape");
  const int smem = (2 * 128 * K + 2 * N * K) * 4;
  VSX_REQUIRE(smem <= 200 * 1024, "umma_selftest: too large");
  VSX_CUDA_TRY(cudaFuncSetAttribute(umma_selftest_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  umma_selftest_kernel<<<1, 128, smem, as_stream(s)>>>(A, B, D, N, K, three);
  VSX_LAUNCH_CHECK("umma_selftest");
  return VSX_OK;
}

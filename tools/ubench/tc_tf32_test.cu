// Standalone check of a hand-written tcgen05.mma kind::tf32 tile on sm_100a:
// D[128 x N] (TMEM, fp32) = A[128 x K] . B[N x K]^T, operands K-major in shared
// memory (SWIZZLE_NONE canonical layout), and the 3xTF32 split
// (a_hi b_hi + a_hi b_lo + a_lo b_hi) against an fp64 host reference.
// Validates the descriptor encodings the GNN kernel would use.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 16;  // K = 2 MMA k-steps of 8 (tf32)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major SWIZZLE_NONE: core matrix = 8 rows x 16 B; element (r, k) at byte
// (r/8)*SBO + (k/4)*LBO + (r%8)*16 + (k%4)*4 with LBO = 128, SBO = (K/4)*128.
__host__ __device__ inline int kmaj_off(int r, int k) {
  return (r / 8) * ((K / 4) * 128) + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version = 1 (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)            // c_format F32
         | (2u << 7)          // a_format TF32
         | (2u << 10)         // b_format TF32
         | (0u << 15)         // a K-major
         | (0u << 16)         // b K-major
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void __launch_bounds__(128) tc_kernel(const float* a, const float* b, float* d,
                                                 int mode, int lbo_sel) {
  __shared__ __align__(128) float sa_hi[M * K], sa_lo[M * K];
  __shared__ __align__(128) float sb_hi[N * K], sb_lo[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // stage operands (split into tf32 hi + lo)
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = a[i], hi = tf32_rna(x), lo = tf32_rna(x - hi);
    sa_hi[kmaj_off(r, k) / 4] = hi;
    sa_lo[kmaj_off(r, k) / 4] = lo;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = b[i], hi = tf32_rna(x), lo = tf32_rna(x - hi);
    sb_hi[kmaj_off(r, k) / 4] = hi;
    sb_lo[kmaj_off(r, k) / 4] = lo;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;"
                 :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t lbo = lbo_sel ? 256u * 0 + ((K / 4) * 128) : 128u;   // lbo_sel=1: swapped
  const uint32_t sbo = lbo_sel ? 128u : (K / 4) * 128;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    int first = 1;
    const int passes = mode == 0 ? 1 : 3;
    for (int pss = 0; pss < passes; ++pss) {
      const float* A = (pss == 2) ? sa_lo : sa_hi;
      const float* B = (pss == 1) ? sb_lo : sb_hi;
      for (int ks = 0; ks < K / 8; ++ks) {  // k-step of 8 tf32 = two 16 B core columns
        const uint64_t da = sdesc(smem_u32(A) + ks * 2 * 128, lbo, sbo);
        const uint64_t db = sdesc(smem_u32(B) + ks * 2 * 128, lbo, sbo);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
            :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(first ? 0 : 1));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(&mbar)));
  }
  // wait for the MMA
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" :: "r"(smem_u32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int row = warp * 32 + lane;
  for (int j = 0; j < N; ++j) d[row * N + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tmem));
}

int main() {
  std::vector<float> a(M * K), b(N * K), d(M * N);
  srand(1);
  for (auto& x : a) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  for (auto& x : b) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  std::vector<double> ref(M * N);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)a[i * K + k] * b[j * K + k];
      ref[i * N + j] = s;
    }
  float *da, *db, *dd;
  cudaMalloc(&da, a.size() * 4); cudaMalloc(&db, b.size() * 4); cudaMalloc(&dd, d.size() * 4);
  cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  for (int lbo_sel = 0; lbo_sel < 2; ++lbo_sel)
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(dd, 0, d.size() * 4);
      tc_kernel<<<1, 128>>>(da, db, dd, mode, lbo_sel);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
      double num = 0, den = 0, mx = 0;
      for (int i = 0; i < M * N; ++i) {
        num += (d[i] - ref[i]) * (d[i] - ref[i]);
        den += ref[i] * ref[i];
        mx = fmax(mx, fabs(d[i] - ref[i]));
      }
      printf("lbo_sel %d mode %s: err=%s relL2 %.3e max %.3e  d[0]=%f ref=%f d[5*N+7]=%f ref=%f\n",
             lbo_sel, mode ? "3xTF32" : "1xTF32", cudaGetErrorString(e), sqrt(num / den), mx,
             d[0], ref[0], d[5 * N + 7], ref[5 * N + 7]);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}

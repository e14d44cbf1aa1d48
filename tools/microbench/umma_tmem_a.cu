// Probe: tcgen05.mma kind::f16 with the A operand in TMEM (written by
// tcgen05.st from registers, thread = row) and B in shared memory (MN-major
// no-swizzle, the layout K7 uses). D[128 x N] = A[128 x K] * B[K x N].
// Tries both packings of two bf16 K-neighbours into a 32-bit TMEM column.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ __forceinline__ uint32_t mn_off(int mn, int k, int MNT) {
  return ((k >> 3) * (MNT >> 3) + (mn >> 3)) * 128 + (k & 7) * 16 + (mn & 7) * 2;
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void probe(const __nv_bfloat16* ga, const __nv_bfloat16* gb, float* gd, int swap_pack, int amaj) {
  __shared__ __align__(1024) unsigned char sb[N * K * 2];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < N * K; e += blockDim.x) {  // gb logical [K][N]
    const int k = e / N, n = e % N;
    *reinterpret_cast<__nv_bfloat16*>(sb + mn_off(n, k, N)) = gb[e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = tmem_base;
  // A -> TMEM columns [64, 64 + K/2): thread (warp q, lane i) = row 32q + i
  {
    const int row = warp * 32 + lane;
    uint32_t r[32];
    for (int c = 0; c < K / 2; ++c) {
      const __nv_bfloat16 lo = ga[row * K + 2 * c], hi = ga[row * K + 2 * c + 1];
      const uint16_t ulo = *reinterpret_cast<const uint16_t*>(&lo), uhi = *reinterpret_cast<const uint16_t*>(&hi);
      r[c] = swap_pack ? ((uint32_t)ulo << 16) | uhi : ((uint32_t)uhi << 16) | ulo;
    }
    const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + 64;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (tid == 0) {
    uint32_t idesc = 0;
    idesc |= 1u << 4;                   // D f32
    idesc |= 1u << 7;                   // A bf16
    idesc |= 1u << 10;                  // B bf16
    idesc |= (uint32_t)amaj << 15;      // a_major
    idesc |= 1u << 16;                  // b_major MN
    idesc |= (uint32_t)(N >> 3) << 17;
    idesc |= (uint32_t)(M >> 4) << 24;
    const uint32_t b_lbo = (N / 8) * 128, b_sbo = 128;
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t bd = make_desc(smem_u32(sb) + kk * 2 * b_lbo, b_lbo, b_sbo);
      const uint32_t ta = tbase + 64 + kk * 8;  // 16 bf16 = 8 columns per K step
      const uint32_t acc = kk > 0 ? 1u : 0u;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tbase),
          "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  {
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t r[16];
      const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 16; ++j) gd[row * N + c0 + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(128));
}

int main() {
  __nv_bfloat16 *ha = new __nv_bfloat16[M * K], *hb = new __nv_bfloat16[K * N];
  float *fa = new float[M * K], *fb = new float[K * N], *ref = new float[M * N], *out = new float[M * N];
  srand(1);
  for (int i = 0; i < M * K; ++i) { fa[i] = (float)((rand() % 17) - 8) / 8.0f; ha[i] = __float2bfloat16(fa[i]); }
  for (int i = 0; i < K * N; ++i) { fb[i] = (float)((rand() % 13) - 6) / 4.0f; hb[i] = __float2bfloat16(fb[i]); }
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)fa[i * K + k] * fb[k * N + j];
      ref[i * N + j] = (float)s;
    }
  __nv_bfloat16 *da, *db;
  float* dd;
  CK(cudaMalloc(&da, M * K * 2));
  CK(cudaMalloc(&db, K * N * 2));
  CK(cudaMalloc(&dd, M * N * 4));
  CK(cudaMemcpy(da, ha, M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, hb, K * N * 2, cudaMemcpyHostToDevice));
  for (int amaj = 0; amaj < 2; ++amaj)
    for (int sw = 0; sw < 2; ++sw) {
      CK(cudaMemset(dd, 0, M * N * 4));
      probe<<<1, 128>>>(da, db, dd, sw, amaj);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("a_major=%d swap=%d: kernel error %s\n", amaj, sw, cudaGetErrorString(e)); return 1; }
      CK(cudaMemcpy(out, dd, M * N * 4, cudaMemcpyDeviceToHost));
      double maxerr = 0;
      for (int i = 0; i < M * N; ++i) maxerr = fmax(maxerr, fabs((double)out[i] - ref[i]));
      printf("A in TMEM, a_major=%d, pack swap=%d: max abs err %.3e (ref[77]=%f out[77]=%f)\n", amaj, sw, maxerr, ref[77], out[77]);
    }
  return 0;
}

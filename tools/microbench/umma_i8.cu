// tcgen05.mma kind::i8 probe (s8/u8 x s8/u8 -> s32, M = 128, K = 32, cta_group::1):
//  1. encoding check: K-major no-swizzle operands in shared memory, both
//     LBO/SBO interpretations, all four signedness combinations, against a
//     CPU product (exact integers);
//  2. A operand from tensor memory (K-major, four K-neighbours per 32-bit column);
//  3. issue rate vs N with A in smem or TMEM: one CTA per SM, one thread
//     issues `iters` MMAs into one accumulator, commit, wait.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8 umma_i8.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// K-major no-swizzle: core matrix = 8 rows x 16 bytes; cores along K `lbo`
// apart, 8-row groups `sbo` apart.
__host__ __device__ inline uint32_t kmaj_off(int row, int k, uint32_t lbo, uint32_t sbo) {
  return (uint32_t)(row >> 3) * sbo + (uint32_t)(k >> 4) * lbo + (uint32_t)(row & 7) * 16 + (uint32_t)(k & 15);
}
__device__ __forceinline__ uint32_t idesc_i8(int M, int N, int as, int bs) {
  uint32_t d = 0;
  d |= 2u << 4;              // D s32
  d |= (uint32_t)as << 7;    // A: 0 u8, 1 s8
  d |= (uint32_t)bs << 10;   // B
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(sa(b)), "r"(ph) : "memory");
}

constexpr int M = 128, K = 64;

// A: [M][K] int8 row-major in global, B: [N][K]; D[M][N] s32
__global__ void check(const int8_t* ga, const int8_t* gb, int* gd, int N, int as, int bs, int swap, int a_tmem) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t lbo = 128, sbo = (K / 16) * 128;  // cores along K contiguous
  unsigned char* a = sm;
  unsigned char* b = sm + M * K;
  for (int e = tid; e < M * K; e += blockDim.x) a[kmaj_off(e / K, e % K, lbo, sbo)] = (unsigned char)ga[e];
  for (int e = tid; e < N * K; e += blockDim.x) b[kmaj_off(e / K, e % K, lbo, sbo)] = (unsigned char)gb[e];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  const uint32_t a_col = 256;  // A in TMEM: columns 256 .. 256 + K/4
  if (a_tmem && warp < 4) {
    // thread = row; column c holds k = 4c .. 4c + 3 (low byte = lowest k)
    const int row = warp * 32 + (tid & 31);
    uint32_t v[16];
    for (int c = 0; c < K / 4; ++c) {
      uint32_t w = 0;
      for (int j = 0; j < 4; ++j) w |= (uint32_t)(unsigned char)ga[row * K + 4 * c + j] << (8 * j);
      v[c] = w;
    }
    const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + a_col;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                 ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (tid == 0) {
    const uint32_t id = idesc_i8(M, N, as, bs);
    for (int kk = 0; kk < K / 32; ++kk) {
      const uint32_t aaddr = sa(a) + kk * 2 * lbo, baddr = sa(b) + kk * 2 * lbo;
      const uint64_t ad = swap ? desc(aaddr, sbo, lbo) : desc(aaddr, lbo, sbo);
      const uint64_t bd = swap ? desc(baddr, sbo, lbo) : desc(baddr, lbo, sbo);
      const uint32_t acc = kk > 0;
      if (a_tmem)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm), "r"(tm + a_col + kk * 8), "l"(bd), "r"(id), "r"(acc));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(ad), "l"(bd), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&bar)));
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (warp < 4) {
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tm + ((uint32_t)(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 8; ++j) gd[row * N + c0 + j] = (int)r[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(512));
}

// issue rate: `iters` MMAs (K = 32 each) over fixed operands
__global__ void rate(int N, int iters, int a_tmem, int ksteps, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (M + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  if (tid == 0) {
    // operands: A 128 x 128 (4 K-steps), B 256 x 128, K-major, LBO 128, SBO 1024
    const uint32_t lbo = 128, sbo = 1024;
    const uint32_t id = idesc_i8(M, N, 1, 0);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int kk = it % ksteps;
      const uint64_t ad = desc(sa(sm) + kk * 2 * lbo, lbo, sbo);
      const uint64_t bd = desc(sa(sm) + M * 128 + kk * 2 * lbo, lbo, sbo);
      if (a_tmem)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm), "r"(tm + 256 + kk * 8), "l"(bd), "r"(id), "r"(1u));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(ad), "l"(bd), "r"(id), "r"(1u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&bar)));
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(512));
}


// rate with `nacc` accumulators used round-robin (128 columns apart) and
// either the no-swizzle layout (sw = 0) or the 128-byte-swizzle K-major
// layout (sw = 1: 8-row x 128-byte atoms, 16-byte chunks XOR row % 8, SBO
// 1024, K advanced by 32 bytes in the start address)
__global__ void rate2(int N, int iters, int nacc, int sw, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (M + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_i8(M, N, 1, 1);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int kk = it & 3, acc = it % nacc;
      uint64_t ad, bd;
      if (sw) {
        ad = desc(sa(sm) + kk * 32, 16, 1024) | (2ull << 61);
        bd = desc(sa(sm) + M * 128 + kk * 32, 16, 1024) | (2ull << 61);
      } else {
        ad = desc(sa(sm) + kk * 2 * 128, 128, 1024);
        bd = desc(sa(sm) + M * 128 + kk * 2 * 128, 128, 1024);
      }
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tm + (uint32_t)(acc * (512 / nacc))), "l"(ad), "l"(bd), "r"(id), "r"(1u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&bar)));
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(512));
}

// swizzle-128 correctness: A [128][128] and B [N][128] int8, K = 128 (4 MMAs)
__global__ void check_sw(const int8_t* ga, const int8_t* gb, int* gd, int N) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  unsigned char* a = sm;
  unsigned char* b = sm + 128 * 128;
  auto off = [](int row, int k) { return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 4) ^ (row & 7)) << 4) | (k & 15))); };
  for (int e = tid; e < 128 * 128; e += blockDim.x) a[off(e / 128, e % 128)] = (unsigned char)ga[e];
  for (int e = tid; e < N * 128; e += blockDim.x) b[off(e / 128, e % 128)] = (unsigned char)gb[e];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, N, 1, 1);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = desc(sa(a) + kk * 32, 16, 1024) | (2ull << 61);
      const uint64_t bd = desc(sa(b) + kk * 32, 16, 1024) | (2ull << 61);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tm), "l"(ad), "l"(bd), "r"(id), "r"((uint32_t)(kk > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&bar)));
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (warp < 4) {
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tm + ((uint32_t)(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 8; ++j) gd[row * N + c0 + j] = (int)r[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(512));
}

int main2() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  CK(cudaFuncSetAttribute(check_sw, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  {
    int8_t *ha = new int8_t[128 * 128], *hb = new int8_t[256 * 128];
    int* out = new int[128 * 256];
    for (int i = 0; i < 128 * 128; ++i) ha[i] = (int8_t)(rand() & 0xFF);
    for (int i = 0; i < 256 * 128; ++i) hb[i] = (int8_t)(rand() & 0xFF);
    int8_t *da, *db; int* dd;
    CK(cudaMalloc(&da, 128 * 128)); CK(cudaMalloc(&db, 256 * 128)); CK(cudaMalloc(&dd, 128 * 256 * 4));
    CK(cudaMemcpy(da, ha, 128 * 128, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, hb, 256 * 128, cudaMemcpyHostToDevice));
    for (int N = 128; N <= 256; N += 128) {
      check_sw<<<1, 128, 64 * 1024>>>(da, db, dd, N);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(out, dd, 128 * N * 4, cudaMemcpyDeviceToHost));
      long long bad = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
          long long r = 0;
          for (int k = 0; k < 128; ++k) r += (long long)ha[i * 128 + k] * hb[j * 128 + k];
          bad += (r != out[i * N + j]);
        }
      printf("check_sw N=%d: mismatches %lld / %d\n", N, bad, 128 * N);
    }
  }
  unsigned long long* dc;
  CK(cudaMalloc(&dc, 8));
  for (int sw = 0; sw < 2; ++sw)
    for (int N = 128; N <= 256; N += 128)
      for (int nacc = 1; nacc <= 4; nacc *= 2) {
        if (N == 256 && nacc == 4) continue;
        const int iters = 4096;
        rate2<<<sms, 128, 64 * 1024>>>(N, iters, nacc, sw, dc);
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        rate2<<<sms, 128, 64 * 1024>>>(N, iters, nacc, sw, dc);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c = 0; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
        printf("rate2 N=%3d nacc=%d %s: %.1f cycles/MMA, %.0f TOPS\n", N, nacc, sw ? "sw128" : "nosw ", (double)c / iters,
               2.0 * M * N * 32 * (double)iters * sms / (ms * 1e-3) / 1e12);
      }
  return 0;
}

// issue-loop overheads: mode bit 0: tcgen05.commit to an mbarrier after every
// MMA; bit 1: tcgen05.fence::after_thread_sync before every MMA; bit 2: an
// mbarrier try_wait (already complete) before every MMA; bit 3: A and B at a
// different 4 KB / 8 KB slot every MMA (16 slots)
__global__ void rate3(int iters, int mode, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bar2, done_bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (16 * 4096 + 8 * 8192) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar2)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&done_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, 256, 1, 1);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (mode & 4) mbar_wait(&bar2, 1);  // parity 1 of a fresh barrier: complete
      if (mode & 2) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int sl = (mode & 8) ? (it & 7) : 0;
      const uint64_t ad = desc(sa(sm) + sl * 4096 + (it & 1) * 256, 128, 256);
      const uint64_t bd = desc(sa(sm) + 16 * 4096 + sl * 8192, 128, 256);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tm + (uint32_t)((it & 1) * 256)), "l"(ad), "l"(bd), "r"(id), "r"(1u));
      if (mode & 1) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&bar)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&done_bar)));
    mbar_wait(&done_bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(512));
}
int main3() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(rate3, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  unsigned long long* dc;
  CK(cudaMalloc(&dc, 8));
  const int modes[8] = {0, 1, 2, 4, 8, 9, 15, 3};
  for (int mi = 0; mi < 8; ++mi) {
    rate3<<<sms, 128, 160 * 1024>>>(2048, modes[mi], dc);
    CK(cudaDeviceSynchronize());
    unsigned long long c = 0;
    CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
    printf("rate3 mode=%2d (commit %d fence %d wait %d slots %d): %.1f cycles/MMA\n", modes[mi], modes[mi] & 1,
           (modes[mi] >> 1) & 1, (modes[mi] >> 2) & 1, (modes[mi] >> 3) & 1, (double)c / 2048);
  }
  return 0;
}

// layout sweep: (LBO, SBO) of K-major no-swizzle operands; K = 32 per MMA
__device__ int g_n = 256;
__global__ void rate4(int iters, int lbo_a, int sbo_a, int lbo_b, int sbo_b, int kstep, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done_bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (160 * 1024) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    reinterpret_cast<uint32_t*>(sm)[i] = (kstep < 0) ? h : 0x01010101u * (i & 3);
  }
  if (kstep < 0) kstep = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&done_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, g_n, 1, 1);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int k = it & 3;
      const uint64_t ad = desc(sa(sm) + k * kstep, lbo_a, sbo_a);
      const uint64_t bd = desc(sa(sm) + 64 * 1024 + k * kstep, lbo_b, sbo_b);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tm + (uint32_t)((it & 1) * 256)), "l"(ad), "l"(bd), "r"(id), "r"(1u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&done_bar)));
    mbar_wait(&done_bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(512));
}
int main4() {
  if (getenv("PROBE4_N")) {
    const int nn = atoi(getenv("PROBE4_N"));
    CK(cudaMemcpyToSymbol(g_n, &nn, sizeof(int)));
    printf("N = %d\n", nn);
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(rate4, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  unsigned long long* dc;
  CK(cudaMalloc(&dc, 8));
  // (lbo, sbo, kstep): kstep = start offset per K-step of 32
  const int cfg[][3] = {{128, 256, 0}, {128, 256, -1}, {128, 256, 0}, {128, 256, -1}, {128, 1024, -1}};
  for (auto& c : cfg) {
    // B (N = 256) with the same pattern, its group stride scaled for 32 groups where SBO spans K
    const int lbo_b = c[0] == 2048 ? 4096 : c[0] == 4096 ? 8192 : c[0] == 256 ? 256 : c[0];
    for (int rep = 0; rep < 3; ++rep) rate4<<<sms, 128, 160 * 1024>>>(8192, c[0], c[1], lbo_b, c[1], c[2], dc);
    CK(cudaDeviceSynchronize());
    unsigned long long cy = 0;
    CK(cudaMemcpy(&cy, dc, 8, cudaMemcpyDeviceToHost));
    printf("rate4 A lbo=%4d sbo=%4d | B lbo=%4d sbo=%4d kstep=%4d (-1: random data): %.1f cycles/MMA\n", c[0], c[1], lbo_b, c[1], c[2],
           (double)cy / 8192);
  }
  return 0;
}

// warp-converged issue loop (all 32 lanes run it, lane 0's MMA enabled):
// mode bit 0: wait on a (complete) mbarrier per MMA, bit 1: the wait loop exits
// on __all_sync, bit 2: tcgen05.commit per MMA, bit 3: ring slot per MMA (16)
__global__ void rate5(int iters, int mode, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[16], done_bar, cbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (192 * 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&done_bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&cbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  if (warp == 0) {
    const uint32_t lead = lane == 0;
    const uint32_t id = idesc_i8(128, 256, 1, 1);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int sl = (mode & 8) ? (it & 15) : 0;
      if (mode & 1) {
        uint32_t done = 0;
        if (mode & 2) {
          do {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(sa(&bar[sl])), "r"(1u) : "memory");
          } while (!__all_sync(0xffffffffu, done));
        } else {
          mbar_wait(&bar[sl], 1);
        }
      }
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint64_t ad = desc(sa(sm) + sl * 4096, 128, 256);
      const uint64_t bd = desc(sa(sm) + 64 * 1024 + sl * 8192, 128, 256);
      asm volatile("{\n.reg .pred p, l;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 l, %5, 0;\n@l tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tm + (uint32_t)((it & 1) * 256)), "l"(ad), "l"(bd), "r"(id), "r"(1u), "r"(lead));
      if (mode & 4)
        asm volatile("{\n.reg .pred l;\nsetp.ne.b32 l, %1, 0;\n@l tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(sa(&cbar)), "r"(lead) : "memory");
    }
    if (lead) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&done_bar)));
      mbar_wait(&done_bar, 0);
      const unsigned long long t1 = clock64();
      if (blockIdx.x == 0) *cyc = t1 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(512));
}
int main5() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(rate5, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024));
  unsigned long long* dc;
  CK(cudaMalloc(&dc, 8));
  const int modes[] = {0, 8, 1, 9, 3, 11, 4, 12, 13, 15};
  for (int md : modes) {
    for (int rep = 0; rep < 2; ++rep) rate5<<<sms, 128, 192 * 1024>>>(4096, md, dc);
    CK(cudaDeviceSynchronize());
    unsigned long long c = 0;
    CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
    printf("rate5 mode=%2d (wait %d all_sync %d commit %d slots %d): %.1f cycles/MMA\n", md, md & 1, (md >> 1) & 1,
           (md >> 2) & 1, (md >> 3) & 1, (double)c / 4096);
  }
  return 0;
}

int main() {
  if (getenv("PROBE5")) return main5();
  if (getenv("PROBE4")) return main4();
  if (getenv("PROBE3")) return main3();
  if (getenv("PROBE2")) return main2();
  int8_t *ha = new int8_t[M * K], *hb = new int8_t[256 * K];
  int* out = new int[M * 256];
  int8_t *da, *db;
  int* dd;
  CK(cudaMalloc(&da, M * K));
  CK(cudaMalloc(&db, 256 * K));
  CK(cudaMalloc(&dd, M * 256 * 4));
  CK(cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  CK(cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  srand(7);
  for (int i = 0; i < M * K; ++i) ha[i] = (int8_t)(rand() & 0xFF);
  for (int i = 0; i < 256 * K; ++i) hb[i] = (int8_t)(rand() & 0xFF);
  CK(cudaMemcpy(da, ha, M * K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, hb, 256 * K, cudaMemcpyHostToDevice));
  const int Ns[3] = {32, 128, 256};
  for (int ni = 0; ni < 3; ++ni)
    for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
      for (int swap = 0; swap < 2; ++swap)
        for (int s = 0; s < 4; ++s) {
          const int N = Ns[ni], as = s & 1, bs = s >> 1;
          if (a_tmem && swap) continue;
          CK(cudaMemset(dd, 0, M * 256 * 4));
          check<<<1, 128, 64 * 1024>>>(da, db, dd, N, as, bs, swap, a_tmem);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("N=%d tmem=%d swap=%d s=%d: %s\n", N, a_tmem, swap, s, cudaGetErrorString(e)); return 1; }
          CK(cudaMemcpy(out, dd, M * N * 4, cudaMemcpyDeviceToHost));
          long long bad = 0;
          for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
              long long r = 0;
              for (int k = 0; k < K; ++k) {
                const int x = as ? (int)ha[i * K + k] : (int)(uint8_t)ha[i * K + k];
                const int y = bs ? (int)hb[j * K + k] : (int)(uint8_t)hb[j * K + k];
                r += (long long)x * y;
              }
              bad += (r != out[i * N + j]);
            }
          printf("check N=%3d a_tmem=%d swap=%d a_signed=%d b_signed=%d: mismatches %lld / %d\n", N, a_tmem, swap, as, bs,
                 bad, M * N);
        }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* dc;
  CK(cudaMalloc(&dc, 8));
  const int Nr[5] = {32, 64, 128, 192, 256};
  for (int ni = 0; ni < 5; ++ni)
    for (int a_tmem = 0; a_tmem < 2; ++a_tmem) {
      const int N = Nr[ni], iters = 4096;
      rate<<<sms, 128, 64 * 1024>>>(N, iters, a_tmem, 4, dc);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      rate<<<sms, 128, 64 * 1024>>>(N, iters, a_tmem, 4, dc);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long c = 0;
      CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
      const double ops = 2.0 * M * N * 32 * (double)iters * sms;
      printf("rate N=%3d A=%s: %.1f cycles/MMA (CTA 0), %.0f TOPS\n", N, a_tmem ? "tmem" : "smem", (double)c / iters,
             ops / (ms * 1e-3) / 1e12);
    }
  return 0;
}

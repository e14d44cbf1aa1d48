// K1z debug harness: runs the gram_f32_ozaki range launches of one plan
// shape directly (the library's own kernel source, debug hook enabled),
// twice, and checks (1) determinism of the per-CTA partials, (2) every digit
// the converters wrote against a host recomputation from A and the recorded
// column exponents, (3) the MMA's span-start flags.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false --expt-relaxed-constexpr \
//     -I include -I paper_2603_11953_b200/csrc tools/oz32_harness.cu -lcuda -o tools/oz32_harness
//   MPSVD_OZ32_STAGES=7x4 ./tools/oz32_harness 22
#define OZ32_DEBUG 1
#include "../paper_2603_11953_b200/csrc/gram_ozaki32.cu"

#include <cmath>
#include <cstring>
#include <vector>

using namespace mpsvd::dev;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double urand() {
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 7;
  rng_state ^= rng_state << 17;
  return ((rng_state >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 22;
  const int nranges = argc > 2 ? atoi(argv[2]) : 16;
  const long long m = 1LL << lg;
  const int n = 128;
  const long long nch = (m + 31) / 32;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int npairs = std::min(sms / 2, gram_ozaki32_max_pairs());
  if (getenv("H_PAIRS")) npairs = atoi(getenv("H_PAIRS"));
  printf("m=2^%d n=%d chunks=%lld pairs=%d ranges=%d\n", lg, n, nch, npairs, nranges);
  std::vector<float> a((size_t)m * n);
  for (size_t i = 0; i < a.size(); i += 2) {
    const double r = sqrt(-2.0 * log(urand())), t = 6.283185307179586 * urand();
    a[i] = (float)(r * cos(t));
    if (i + 1 < a.size()) a[i + 1] = (float)(r * sin(t));
  }
  float* d_a;
  CK(cudaMalloc(&d_a, a.size() * 4));
  CK(cudaMemcpy(d_a, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
  double2* d_part;
  const size_t pbytes = gram_ozaki32_partial_bytes(npairs);
  CK(cudaMalloc(&d_part, pbytes));
  int* d_bad;
  CK(cudaMalloc(&d_bad, 128 * 4));
  Oz32Dbg dbg = {};
  CK(cudaMalloc(&dbg.digits, (size_t)nch * 6 * 128 * 32));
  CK(cudaMalloc(&dbg.E, (size_t)nch * 128 * 2));
  CK(cudaMalloc(&dbg.fresh, (size_t)nch * 2 * 4));
  std::vector<long long> bounds;
  {
    const long long base = m / nranges, extra = m % nranges;
    long long row = 0;
    for (int b = 0; b < nranges; ++b) {
      bounds.push_back(row / 32);
      row += base + (b < extra ? 1 : 0);
    }
    bounds.push_back(nch);
  }
  const int pch = 400;
  dbg.prof_chunks = pch;
  CK(cudaMalloc(&dbg.prof, (size_t)2 * pch * 12 * 8));
  CK(cudaMemset(dbg.prof, 0, (size_t)2 * pch * 12 * 8));
  std::vector<double2> p0(pbytes / 16), p1(pbytes / 16);
  std::vector<int8_t> dig((size_t)nch * 6 * 128 * 32);
  std::vector<short> E((size_t)nch * 128);
  std::vector<int> fr((size_t)nch * 2);
  for (int run = 0; run < 3; ++run) {
    Oz32Dbg d2 = dbg;
    if (getenv("H_NODIG")) d2.digits = nullptr, d2.E = nullptr;
    CK(cudaMemcpyToSymbol(g_oz32_dbg, &d2, sizeof(d2)));
    CK(cudaMemset(dbg.digits, 0x55, (size_t)nch * 6 * 128 * 32));
    CK(cudaMemset(d_bad, 0, 128 * 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int b = 0; b < nranges; ++b)
      CK(launch_gram_ozaki32_range(d_a, m, m, n, bounds[b], bounds[b + 1], npairs, d_part, d_bad, b > 0, 0));
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<double2>& p = run == 0 ? p0 : p1;
    CK(cudaMemcpy(p.data(), d_part, pbytes, cudaMemcpyDeviceToHost));
    long long ndiff = 0;
    int first_cta = -1;
    if (run > 0)
      for (size_t i = 0; i < p0.size(); ++i)
        if (memcmp(&p0[i], &p1[i], 16)) {
          if (first_cta < 0) first_cta = (int)(i / (128 * 128));
          ++ndiff;
        }
    printf("run %d: %.3f ms (debug stores on), partial entries differing from run 0: %lld (first CTA %d)\n", run, ms,
           ndiff, first_cta);
    // digits vs host
    CK(cudaMemcpy(dig.data(), dbg.digits, dig.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(E.data(), dbg.E, E.size() * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(fr.data(), dbg.fresh, fr.size() * 4, cudaMemcpyDeviceToHost));
    long long bad = 0, shown = 0;
    for (long long ch = 0; ch < (getenv("H_NODIG") ? 0 : nch); ++ch)
      for (int c = 0; c < n; ++c) {
        const int e = E[ch * 128 + c];
        for (int r = 0; r < 32; ++r) {
          const long long row = ch * 32 + r;
          uint32_t bits = 0;
          if (row < m) memcpy(&bits, &a[(size_t)c * m + row], 4);
          const unsigned long long y = fixed48(bits, e);
          for (int pp = 1; pp <= 6; ++pp) {
            const int8_t want = (int8_t)(((y >> (8 * (6 - pp))) & 0xFF) ^ 0x80);
            const int8_t got = dig[((ch * 6 + pp - 1) * 128 + c) * 32 + r];
            if (want != got) {
              ++bad;
              if (pp == 1 && shown++ < 12) {
                // which chunk's value did the converter see? the same (column, row) of chunk ch + d, d in [-16, 16]
                int hit = 99;
                for (int d = -16; d <= 16 && hit == 99; ++d) {
                  const long long c2 = ch + d;
                  if (c2 < 0 || c2 >= nch || d == 0) continue;
                  uint32_t b2 = 0;
                  if (c2 * 32 + r < m) memcpy(&b2, &a[(size_t)c * m + c2 * 32 + r], 4);
                  const unsigned long long y2 = fixed48(b2, e);
                  bool all = true;
                  for (int q2 = 1; q2 <= 6; ++q2)
                    all &= (int8_t)(((y2 >> (8 * (6 - q2))) & 0xFF) ^ 0x80) == dig[((ch * 6 + q2 - 1) * 128 + c) * 32 + r];
                  if (all) hit = d;
                }
                // position of chunk ch in its pair's share of its range
                int rb = 0;
                while (rb + 1 < (int)bounds.size() - 1 && bounds[rb + 1] <= ch) ++rb;
                const long long nall = bounds[rb + 1] - bounds[rb];
                int pr = 0;
                while (pr + 1 < npairs && bounds[rb] + nall * (pr + 1) / npairs <= ch) ++pr;
                const long long jpos = ch - (bounds[rb] + nall * pr / npairs);
                printf("  mismatch chunk %lld (range %d pair %d j %lld) col %d row %d: seen value = chunk offset %d\n", ch,
                       rb, pr, jpos, c, r, hit);
              }
            }
          }
        }
      }
    if (run == 0) {
      // pipeline timing of pair 0 over its first range (SM clock cycles): per event the mean gap to the
      // previous event of the same chunk, and the mean chunk period of each event stream
      std::vector<unsigned long long> pr((size_t)2 * pch * 12);
      CK(cudaMemcpy(pr.data(), dbg.prof, pr.size() * 8, cudaMemcpyDeviceToHost));
      const char* names[12] = {"tma issue", "scouts done", "conv: slot free", "conv: half done", "copier issue",
                               "mma: slot full", "mma: committed", "conv: A in regs", "conv: iter start",
                               "conv: meta ok", "conv: a_full ok", "conv: released"};
      const long long nj = std::min<long long>(pch, bounds[1] / npairs);
      for (int gg = 0; gg < 2; ++gg) {
        printf("  CTA %d of pair 0, chunks 20..%lld:\n", gg, nj - 1);
        for (int ev = 0; ev < 12; ++ev) {
          double per = 0, lag = 0;
          long long cnt = 0;
          for (long long j = 21; j < nj; ++j) {
            const unsigned long long* r = &pr[((size_t)gg * pch + j) * 12];
            const unsigned long long* r0 = &pr[((size_t)gg * pch + j - 1) * 12];
            per += (double)(r[ev] - r0[ev]);
            lag += (double)r[ev] - (double)r[0];
            ++cnt;
          }
          printf("    %-16s period %8.1f cyc   after tma issue %9.1f cyc\n", names[ev], per / cnt, lag / cnt);
        }
      }
    }
    long long fmis = 0;
    for (long long ch = 0; ch < nch; ++ch)
      if (fr[2 * ch] != fr[2 * ch + 1]) ++fmis;
    long long nfresh = 0;
    for (long long ch = 0; ch < nch; ++ch) nfresh += fr[2 * ch];
    printf("  digit mismatches: %lld; fresh flags differing between the pair's CTAs: %lld; span starts: %lld\n", bad,
           fmis, nfresh);
  }
  return 0;
}

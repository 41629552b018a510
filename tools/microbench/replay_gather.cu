// Gather roof of a REAL column sequence: replays a matrix's col_idx (CSR order, the order the
// streaming kernel consumes a unit's row-major list) as pure B-row gathers -- no list reads from
// HBM, no FMAs that wait on a row end, no C stores -- so the time is what the B-row gathers alone
// cost on this access pattern (its L2 hit rate, its HBM misses), the floor for k_spmm_stream.
//
// Work is split like the SpMM's: warps claim contiguous segments of SEG entries from a global
// counter (one unit ~ 150 nonzeros on R-MAT); a lane loads 16 B of each of R rows in flight.
// Orders: "csr" (as given), "shuffled" (same multiset, random order: no temporal locality),
// "sorted" (ascending column: every row fetched from HBM once, then L1/L2 reuse).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o replay_gather replay_gather.cu
//   ./replay_gather cols.i32 n_cols row_bytes
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int SEG = 160;

// SETUP = dependent global loads each warp waits for at every segment start (the streaming
// kernel's unit setup: descriptor -> group row/slot -> bitmaps -> list copy), chased through
// `chain` (an L2-resident permutation) before the segment's first gathers are issued.
template <int R, int RB, int SETUP = 0>
__global__ void __launch_bounds__(256) k_replay(const char* __restrict__ B, const int* __restrict__ idx, long n,
                                                unsigned* counter, float* out, const int* __restrict__ chain = nullptr,
                                                int seg = SEG) {
  constexpr int LPR = RB / 16;   // lanes per row
  constexpr int RPI = 32 / LPR;  // rows per warp instruction
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  const long nseg = (n + seg - 1) / seg;
  int link = threadIdx.x;
  for (;;) {
    unsigned s = 0;
    if (lane == 0) s = atomicAdd(counter, 1u);
    s = __shfl_sync(0xffffffffu, s, 0);
    if ((long)s >= nseg) break;
#pragma unroll 1
    for (int k = 0; k < SETUP; ++k) link = __ldcg(chain + ((link + s) & 1048575));
    if (link == -7) out[1] = 0.f;
    const long e0 = (long)s * seg, e1 = min(n, e0 + seg);
    for (long base = e0; base < e1; base += (long)R * RPI) {
      int r[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const long i = base + (long)k * RPI + lane / LPR;
        r[k] = i < e1 ? __ldg(idx + i) : -1;
      }
      uint4 v[R];
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (r[k] >= 0) v[k] = __ldg(reinterpret_cast<const uint4*>(B + (long)r[k] * RB + (lane % LPR) * 16));
        else v[k] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < R; ++k)
        acc += __int_as_float(v[k].x) + __int_as_float(v[k].y) + __int_as_float(v[k].z) + __int_as_float(v[k].w);
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  if (argc < 4) {
    printf("usage: %s cols.i32 n_cols row_bytes\n", argv[0]);
    return 2;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 2;
  fseek(f, 0, SEEK_END);
  const long n = ftell(f) / 4;
  fseek(f, 0, SEEK_SET);
  std::vector<int> h(n);
  if (fread(h.data(), 4, n, f) != (size_t)n) return 2;
  fclose(f);
  const long n_cols = atol(argv[2]);
  const int RB = atoi(argv[3]);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char* B;
  CK(cudaMalloc(&B, (size_t)n_cols * RB));
  {
    std::vector<uint32_t> hb((size_t)n_cols * RB / 4);
    std::mt19937 rb(11);
    for (auto& x : hb) x = 0x3f000000u | (rb() & 0x7fffffu);  // floats in [0.5, 1)
    CK(cudaMemcpy(B, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
  }
  int* idx;
  CK(cudaMalloc(&idx, n * 4));
  unsigned* counter;
  CK(cudaMalloc(&counter, 4));
  float* out;
  CK(cudaMalloc(&out, 8));
  // flush buffer: 512 MB written between timed launches so no run inherits the last one's L2
  char* flush;
  const size_t flush_bytes = 512ull << 20;
  CK(cudaMalloc(&flush, flush_bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("entries %ld, B %ld rows x %d B (%.0f MB), gathered %.2f GB per launch\n", n, n_cols, RB,
         n_cols * (double)RB / 1e6, n * (double)RB / 1e9);
  auto timeit = [&](auto launch) {
    std::vector<float> ts;
    for (int it = 0; it < 6; ++it) {
      CK(cudaMemset(flush, it, flush_bytes));
      CK(cudaMemset(counter, 0, 4));
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it) ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
  };
  std::vector<int> order = h;
  for (const char* name : {"csr", "shuffled", "sorted"}) {
    if (name[0] == 's' && name[1] == 'h') {
      std::mt19937_64 rng(3);
      std::shuffle(order.begin(), order.end(), rng);
    } else if (name[0] == 's') {
      std::sort(order.begin(), order.end());
    }
    CK(cudaMemcpy(idx, order.data(), n * 4, cudaMemcpyHostToDevice));
    auto run = [&](auto kern, int ctas, const char* rname) {
      const float ms = timeit([&] { kern<<<sms * ctas, 256>>>(B, idx, n, counter, out, nullptr, SEG); });
      printf("  %-8s %-3s ctas/SM %d: %.3f ms  %7.0f GB/s gathered\n", name, rname, ctas, ms, n * (double)RB / ms / 1e6);
    };
    for (int c : {4, 6, 8}) {
      if (RB == 512) {
        run(k_replay<6, 512>, c, "R6");
        run(k_replay<8, 512>, c, "R8");
      } else {
        run(k_replay<6, 256>, c, "R6");
        run(k_replay<8, 256>, c, "R8");
      }
    }
    if (name[0] == 'c') {  // L1 capacity: the same gathers with the streaming kernel's 23 KB of
                           // shared memory per CTA (and twice that) taken from the L1 carve-out
      for (int kb : {23, 46}) {
        auto run3 = [&](auto kern) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024));
          const float ms = timeit([&] { kern<<<sms * 4, 256, kb * 1024>>>(B, idx, n, counter, out, nullptr, SEG); });
          printf("  csr      R6  ctas/SM 4 smem %2d KB/CTA: %.3f ms\n", kb, ms);
        };
        if (RB == 512) run3(k_replay<6, 512>);
        else run3(k_replay<6, 256>);
      }
    }
    if (name[0] == 'c') {  // unit-setup cost: dependent loads per segment, and longer segments
      int* chain;
      CK(cudaMalloc(&chain, 4 << 20));
      std::vector<int> hc(1 << 20);
      std::mt19937_64 rng(5);
      for (int i = 0; i < (1 << 20); ++i) hc[i] = (int)(rng() & 1048575);
      CK(cudaMemcpy(chain, hc.data(), 4 << 20, cudaMemcpyHostToDevice));
      for (int seg : {160, 640}) {
        auto run2 = [&](auto kern, const char* rname) {
          const float ms = timeit([&] { kern<<<sms * 4, 256>>>(B, idx, n, counter, out, chain, seg); });
          printf("  csr      R6  ctas/SM 4 seg %4d %-9s: %.3f ms\n", seg, rname, ms);
        };
        if (RB == 512) {
          run2(k_replay<6, 512, 0>, "setup 0");
          run2(k_replay<6, 512, 2>, "setup 2");
          run2(k_replay<6, 512, 4>, "setup 4");
        } else {
          run2(k_replay<6, 256, 0>, "setup 0");
          run2(k_replay<6, 256, 2>, "setup 2");
          run2(k_replay<6, 256, 4>, "setup 4");
        }
      }
      cudaFree(chain);
    }
    fflush(stdout);
  }
  return 0;
}

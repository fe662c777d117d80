// Microbenchmark: CUB onesweep with wider radix digits for the 28-bit box keys.
// 8-bit digits (CUB's sm_100 default) take 4 passes over 28 bits; 10- or
// 11-bit digits take 3.  Checks the outputs are identical and times each.
// Measured on B200 (1e8 random 28-bit keys + u32 values): default 2.47 ms,
// 10-bit 256x16 3.69 ms, 10-bit 256x24 3.61 ms (identical output) -- the
// wider-digit ranking costs more than the saved pass; 192x30 did not finish.
// 11-bit tiles do not fit 48 KB of static shared memory.  Not adopted.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/sort_digits_bench.cu -o /tmp/sdb
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>

using Key = uint32_t;
using Val = uint32_t;
using Off = int;

template <int BITS, int THREADS, int ITEMS>
struct Hub {
  using Base = typename cub::detail::radix::policy_hub<Key, Val, Off>::Policy1000;
  struct Policy : cub::ChainedPolicy<1000, Policy, Policy> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = BITS;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, Key, BITS>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, BITS>;
    using OnesweepPolicy = cub::AgentRadixSortOnesweepPolicy<
        THREADS, ITEMS, Key, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
        cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, BITS>;
    using ScanPolicy = typename Base::ScanPolicy;
    using DownsweepPolicy = typename Base::DownsweepPolicy;
    using AltDownsweepPolicy = typename Base::AltDownsweepPolicy;
    using UpsweepPolicy = typename Base::UpsweepPolicy;
    using AltUpsweepPolicy = typename Base::AltUpsweepPolicy;
    using SingleTilePolicy = typename Base::SingleTilePolicy;
    using SegmentedPolicy = typename Base::SegmentedPolicy;
    using AltSegmentedPolicy = typename Base::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy;
};

template <typename H>
float run(const Key* kin, Key* kout, const Val* vin, Val* vout, int n, int end_bit, void*& tmp,
          size_t& tmp_cap, int reps) {
  cub::DoubleBuffer<Key> kb(const_cast<Key*>(kin), kout);
  cub::DoubleBuffer<Val> vb(const_cast<Val*>(vin), vout);
  size_t need = 0;
  cub::DispatchRadixSort<false, Key, Val, Off, H>::Dispatch(nullptr, need, kb, vb, n, 0, end_bit,
                                                            false, 0);
  if (need > tmp_cap) { cudaFree(tmp); cudaMalloc(&tmp, need); tmp_cap = need; }
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cub::DoubleBuffer<Key> k2(const_cast<Key*>(kin), kout);
    cub::DoubleBuffer<Val> v2(const_cast<Val*>(vin), vout);
    cudaEventRecord(a);
    cudaError_t e = cub::DispatchRadixSort<false, Key, Val, Off, H>::Dispatch(
        tmp, need, k2, v2, n, 0, end_bit, false, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  return best;
}

__global__ void init(Key* k, Val* v, int n, uint32_t mask) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    k[i] = (uint32_t)x & mask;
    v[i] = i;
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int n = 100000000, end_bit = 28;
  Key *k, *ko, *kref; Val *v, *vo, *vref;
  cudaMalloc(&k, n * 4); cudaMalloc(&ko, n * 4); cudaMalloc(&kref, n * 4);
  cudaMalloc(&v, n * 4); cudaMalloc(&vo, n * 4); cudaMalloc(&vref, n * 4);
  init<<<(n + 255) / 256, 256>>>(k, v, n, (1u << end_bit) - 1);
  void* tmp = nullptr; size_t cap = 0;
  using Def = cub::detail::radix::policy_hub<Key, Val, Off>;
  float t8 = run<Def>(k, kref, v, vref, n, end_bit, tmp, cap, 6);
  printf("default (8-bit, 4 passes): %.3f ms\n", t8);
  std::vector<uint32_t> hk(n), hv(n), rk(n), rv(n);
  cudaMemcpy(rk.data(), kref, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(rv.data(), vref, n * 4, cudaMemcpyDeviceToHost);
  auto check = [&](const char* name, float t) {
    cudaMemcpy(hk.data(), ko, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hv.data(), vo, n * 4, cudaMemcpyDeviceToHost);
    printf("%s: %.3f ms, identical=%d\n", name, t, (int)(hk == rk && hv == rv));
  };
  check("10-bit 256x16", run<Hub<10, 256, 16>>(k, ko, v, vo, n, end_bit, tmp, cap, 6));
  check("10-bit 256x24", run<Hub<10, 256, 24>>(k, ko, v, vo, n, end_bit, tmp, cap, 6));
  check("9-bit 384x23 (4 passes)", run<Hub<9, 384, 23>>(k, ko, v, vo, n, end_bit, tmp, cap, 6));
  check("8-bit 384x23 (same as default)", run<Hub<8, 384, 23>>(k, ko, v, vo, n, end_bit, tmp, cap, 6));
  return 0;
}

// host_policy.cpp — host-side control plane of the GRASS hot path:
// counter-based RNG, Eq. 3 softmax, the gamma-of-N_L sampler, shard ranges
// and the schedule.  Compiled with -ffp-contract=off so every fp64 operation
// rounds exactly as written (the sampler's bit-exact contract).
//
// Independent of oracle/: written from PAPER.md and the DESIGN.md readings.
#include <cmath>
#include <cstdint>
#include <vector>

#include "grass_internal.h"

namespace grass {

// Standard SplitMix64 output function (R7).
uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Counter-based uniform in [0,1) for draw k of sampling period `period` (R7).
double uniform01(uint64_t seed, uint64_t period, uint32_t k) {
  const uint64_t key = splitmix64(seed);
  const uint64_t ctr = (period << 16) + (uint64_t)k;
  return (double)(splitmix64(key ^ ctr) >> 11) * 0x1.0p-53;
}

// Eq. 3 with reading R3: optional max-normalisation
// m~ = m / max m (m == 0 -> m~ = 0), then p_l = exp((m~_l - max m~)/tau) / sum.
// The denominator is the ascending sequential fp64 sum.
bool softmax_probs(const double* m, int n, double tau, bool normalize, double* p) {
  if (n <= 0 || !(tau > 0.0)) return false;
  std::vector<double> mt(m, m + n);
  if (normalize) {
    double M = mt[0];
    for (int i = 1; i < n; ++i) M = mt[i] > M ? mt[i] : M;
    for (int i = 0; i < n; ++i) mt[i] = M > 0.0 ? mt[i] / M : 0.0;
  }
  double mx = mt[0];
  for (int i = 1; i < n; ++i) mx = mt[i] > mx ? mt[i] : mx;
  double tot = 0.0;
  for (int i = 0; i < n; ++i) {
    p[i] = std::exp((mt[i] - mx) / tau);
    tot += p[i];
  }
  for (int i = 0; i < n; ++i) p[i] = p[i] / tot;
  return true;
}

// "samples gamma layers out of N_L", reading R6: gamma
// sequential draws without replacement, each proportional to p over the
// still-available layers (renormalised), ascending walk with strict x < c,
// fallback to the last available layer.  Output in draw order.
bool sample_from_probs(const double* p, int n, int gamma, uint64_t seed, uint64_t period,
                       int32_t* ids) {
  if (n <= 0 || gamma < 1 || gamma > n) return false;
  std::vector<int32_t> avail(n);
  for (int i = 0; i < n; ++i) avail[i] = i;
  for (int k = 0; k < gamma; ++k) {
    const double u = uniform01(seed, period, (uint32_t)k);
    double R = 0.0;
    for (int32_t l : avail) R += p[l];
    const double x = u * R;
    double c = 0.0;
    size_t pick = avail.size() - 1;
    for (size_t j = 0; j < avail.size(); ++j) {
      c += p[avail[j]];
      if (x < c) {
        pick = j;
        break;
      }
    }
    ids[k] = avail[pick];
    avail.erase(avail.begin() + (long)pick);
  }
  return true;
}

bool shard_range(int64_t numel, int world, int rank, int64_t* off, int64_t* cnt) {
  if (numel < 1 || world < 1 || rank < 0 || rank >= world) return false;
  if (world == 1) {
    *off = 0;
    *cnt = numel;
    return true;
  }
  if (numel % (4 * (int64_t)world) != 0) return false;
  const int64_t s = numel / world;
  *off = s * rank;
  *cnt = s;
  return true;
}

// PAPER.md:111-121 with R11 (T_u a multiple of T_s).
int schedule_decision(int64_t step, int T_p, int T_s, int T_u) {
  if (T_u <= 0) T_u = T_s;
  if (step < T_p) return GRASS_DECIDE_PROBE;
  const int64_t d = step - T_p;
  if (d == 0 || d % T_u == 0) return GRASS_DECIDE_COMMIT_RESAMPLE;
  if (d % T_s == 0) return GRASS_DECIDE_RESAMPLE;
  return GRASS_DECIDE_CONTINUE;
}

}  // namespace grass

// bank_gen.cpp — native kernel-bank generation.
//
// The reference draws its bank on the host from numpy's
// Generator(Philox(key=seed)) in a fixed per-kernel order
// (kernels.py:243-308) — about 28 us of Python per kernel, 2.8 s at 100k
// kernels.  This file replays the same stream in C++: the same draws in the
// same order through re-implementations of the numpy 2.x algorithms the
// reference calls (numpy is a pinned third-party dependency, 2.3.5 here):
//
//   Philox4x64-10 bit generator, counter incremented before each block of
//     four outputs, key = (seed, 0); next_uint32 hands out the low then the
//     high half of one 64-bit output;
//   Generator.integers(0, 3)   -> Lemire's bounded 32-bit method;
//   Generator.uniform / random -> low + (high - low) * ((u64 >> 11) * 2^-53);
//   Generator.standard_normal  -> 256-level ziggurat (tables: ziggurat.h);
//   Generator.choice(C, m, replace=False) -> Floyd's algorithm with a
//     linear-probing set (tail shuffle for C > 10000, m > C / 50), then a
//     Fisher-Yates shuffle of the picks; the reference sorts them;
//   ndarray.mean               -> numpy's pairwise sum / n.
//
// Bit-identity with numpy is pinned by tests/test_bank_native.py (every
// field of the bank, many shapes and seeds) and by the golden reference
// fingerprints (tests/golden/banks.json).  Values that numpy computes with
// its own vectorised log2 (the dilation and channel-count exponent bounds)
// are passed in from Python.  Compiled with -ffp-contract=off.
#include "../../include/rocket_b200.h"
#include "rk_internal.h"
#include "ziggurat.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

namespace {

class Philox {
 public:
  explicit Philox(uint64_t seed) : key_{seed, 0} {}

  uint64_t next64() {
    if (pos_ < 4) return buf_[pos_++];
    if (++ctr_[0] == 0 && ++ctr_[1] == 0 && ++ctr_[2] == 0) ++ctr_[3];
    block();
    pos_ = 1;
    return buf_[0];
  }
  uint32_t next32() {
    if (has32_) {
      has32_ = false;
      return half_;
    }
    const uint64_t v = next64();
    has32_ = true;
    half_ = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }

 private:
  void block() {
    uint64_t c0 = ctr_[0], c1 = ctr_[1], c2 = ctr_[2], c3 = ctr_[3];
    uint64_t k0 = key_[0], k1 = key_[1];
    for (int round = 0; round < 10; ++round) {
      if (round) {
        k0 += 0x9E3779B97F4A7C15ull;
        k1 += 0xBB67AE8584CAA73Bull;
      }
      const unsigned __int128 p0 = (unsigned __int128)0xD2E7470EE14C6C93ull * c0;
      const unsigned __int128 p1 = (unsigned __int128)0xCA5A826395121157ull * c2;
      const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
      const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
      c0 = hi1 ^ c1 ^ k0;
      c1 = lo1;
      c2 = hi0 ^ c3 ^ k1;
      c3 = lo0;
    }
    buf_[0] = c0;
    buf_[1] = c1;
    buf_[2] = c2;
    buf_[3] = c3;
  }

  uint64_t ctr_[4] = {0, 0, 0, 0};
  uint64_t key_[2];
  uint64_t buf_[4] = {0, 0, 0, 0};
  int pos_ = 4;
  bool has32_ = false;
  uint32_t half_ = 0;
};

// Generator.integers(0, rng + 1) for rng < 2^32 - 1 (numpy's
// random_bounded_uint64 -> Lemire's method on 32-bit draws).
uint64_t bounded(Philox& g, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFull) return g.next32();
  const uint32_t excl = (uint32_t)rng + 1u;
  uint64_t m = (uint64_t)g.next32() * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t threshold = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
    while (left < threshold) {
      m = (uint64_t)g.next32() * excl;
      left = (uint32_t)m;
    }
  }
  return m >> 32;
}

uint64_t bounded64(Philox& g, uint64_t rng) {
  if (rng <= 0xFFFFFFFFull) return bounded(g, rng);
  // 64-bit Lemire (populations beyond 2^32 never occur for channel counts)
  const uint64_t excl = rng + 1;
  unsigned __int128 m = (unsigned __int128)g.next64() * excl;
  uint64_t left = (uint64_t)m;
  if (left < excl) {
    const uint64_t threshold = (0xFFFFFFFFFFFFFFFFull - rng) % excl;
    while (left < threshold) {
      m = (unsigned __int128)g.next64() * excl;
      left = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

double uniform(Philox& g, double low, double high) {
  const double range = high - low;
  return low + range * g.next_double();
}

double standard_normal(Philox& g) {
  for (;;) {
    uint64_t r = g.next64();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * rk_zig::wi[idx];
    if (sign & 0x1) x = -x;
    if (rabs < rk_zig::ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = -rk_zig::kInvR * std::log1p(-g.next_double());
        const double yy = -std::log1p(-g.next_double());
        if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(rk_zig::kR + xx) : rk_zig::kR + xx;
      }
    }
    if (((rk_zig::fi[idx - 1] - rk_zig::fi[idx]) * g.next_double() + rk_zig::fi[idx]) < std::exp(-0.5 * x * x))
      return x;
  }
}

uint64_t gen_mask(uint64_t v) {
  for (int s = 1; s <= 32; s <<= 1) v |= v >> s;
  return v;
}

// Generator.choice(pop, size, replace=False) (shuffle=True).
void choice_without_replacement(Philox& g, int64_t pop, int64_t size, std::vector<int64_t>& out) {
  out.assign((size_t)size, 0);
  if (pop > 10000 && size > pop / 50) {
    // tail shuffle of arange(pop)
    std::vector<int64_t> idx((size_t)pop);
    for (int64_t i = 0; i < pop; ++i) idx[(size_t)i] = i;
    const int64_t first = std::max<int64_t>(pop - size, 1);
    for (int64_t i = pop - 1; i >= first; --i) {
      const int64_t j = (int64_t)bounded64(g, (uint64_t)i);
      std::swap(idx[(size_t)i], idx[(size_t)j]);
    }
    std::copy(idx.end() - size, idx.end(), out.begin());
    return;
  }
  // Floyd's algorithm with an open-addressing set
  const uint64_t mask = gen_mask((uint64_t)(1.2 * (double)size));
  std::vector<uint64_t> set((size_t)(mask + 1), ~0ull);
  for (int64_t j = pop - size; j < pop; ++j) {
    const uint64_t val = bounded64(g, (uint64_t)j);
    uint64_t loc = val & mask;
    while (set[loc] != ~0ull && set[loc] != val) loc = (loc + 1) & mask;
    if (set[loc] == ~0ull) {
      set[loc] = val;
      out[(size_t)(j - pop + size)] = (int64_t)val;
    } else {
      loc = (uint64_t)j & mask;
      while (set[loc] != ~0ull) loc = (loc + 1) & mask;
      set[loc] = (uint64_t)j;
      out[(size_t)(j - pop + size)] = j;
    }
  }
  for (int64_t i = size - 1; i >= 1; --i) {
    const int64_t j = (int64_t)bounded64(g, (uint64_t)i);
    std::swap(out[(size_t)i], out[(size_t)j]);
  }
}

// numpy's pairwise summation (add.reduce over a contiguous float64 array).
double pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

}  // namespace

extern "C" int rk_generate_bank(int64_t count, int32_t l_series, int32_t n_channels, uint64_t seed,
                                int32_t center_weights, const double* exponent_bounds, double channel_bound,
                                int32_t* lengths, double* biases, int32_t* dilations, int32_t* paddings,
                                int32_t* channel_counts, int32_t* channel_indices, int64_t index_capacity,
                                double* weights, int64_t weight_capacity, int64_t* n_weights,
                                int64_t* n_indices) {
  static const int kLengths[3] = {7, 9, 11};
  if (count < 1 || l_series < 11 || n_channels < 1)
    return rk_set_error(RK_ERR_INVALID, "count >= 1, l_series >= 11 and n_channels >= 1 are required");
  if (!exponent_bounds || !lengths || !biases || !dilations || !paddings || !channel_counts || !channel_indices ||
      !weights || !n_weights || !n_indices)
    return rk_set_error(RK_ERR_INVALID, "NULL argument");
  Philox g(seed);
  std::vector<int64_t> picks;
  // the variable-length streams are drawn into exact-size buffers, then
  // copied out; a caller buffer that is too small gets RK_ERR_CAPACITY with
  // the sizes needed in *n_weights / *n_indices (the caller can size its
  // buffers from an estimate and retry: the draw is deterministic)
  std::vector<int32_t> idx;
  std::vector<double> wts;
  idx.reserve((size_t)count);
  wts.reserve((size_t)count * 11);
  for (int64_t k = 0; k < count; ++k) {
    const int li = (int)bounded(g, 2);
    const int lk = kLengths[li];
    int64_t nsel = 1;
    if (n_channels > 1) {
      const double u = uniform(g, 0.0, channel_bound);
      nsel = std::min<int64_t>(std::max<int64_t>((int64_t)std::pow(2.0, u), 1), n_channels);
      choice_without_replacement(g, n_channels, nsel, picks);
      std::sort(picks.begin(), picks.end());
      for (int64_t c = 0; c < nsel; ++c) idx.push_back((int32_t)picks[(size_t)c]);
    } else {
      idx.push_back(0);
    }
    const int64_t nw = nsel * lk;
    const size_t w0 = wts.size();
    for (int64_t j = 0; j < nw; ++j) wts.push_back(standard_normal(g));
    double* w = wts.data() + w0;
    if (center_weights) {
      const double mean = pairwise_sum(w, nw) / (double)nw;
      for (int64_t j = 0; j < nw; ++j) w[j] = w[j] - mean;
    }
    const double bias = uniform(g, -1.0, 1.0);
    const int32_t d = (int32_t)std::pow(2.0, uniform(g, 0.0, exponent_bounds[li]));
    const int32_t p = g.next_double() < 0.5 ? (lk - 1) * d / 2 : 0;
    lengths[k] = lk;
    biases[k] = bias;
    dilations[k] = d;
    paddings[k] = p;
    channel_counts[k] = (int32_t)nsel;
  }
  *n_weights = (int64_t)wts.size();
  *n_indices = (int64_t)idx.size();
  if ((int64_t)idx.size() > index_capacity || (int64_t)wts.size() > weight_capacity)
    return rk_set_error(RK_ERR_CAPACITY, "channel index / weight buffer too small (sizes needed in n_indices / n_weights)");
  std::memcpy(channel_indices, idx.data(), idx.size() * sizeof(int32_t));
  std::memcpy(weights, wts.data(), wts.size() * sizeof(double));
  return RK_OK;
}

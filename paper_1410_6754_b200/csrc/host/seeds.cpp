// Seeded sample streams of the reference, restated natively.
//
// Reference: SeedSpec (core.py:46-71) names a stream by
//   blake2b(f"{master}\x1f{stream_id}\x1f", digest_size=16)  (core.py:62-64)
// and seeds CPython's random.Random with the big-endian integer of that
// digest (core.py:66-67).  draw_sample (ams.py:157-175) then takes
//   sorted(rng.sample(range(len), take))                      (ams.py:171-173)
//
// The pieces restated here are the published algorithms those calls run:
//   * BLAKE2b (RFC 7693), unkeyed, 16-byte digest;
//   * MT19937 with CPython's init_by_array seeding of an int (its 32-bit
//     little-endian words, leading zero words dropped) and genrand tempering;
//   * CPython 3.12 Random._randbelow_with_getrandbits and Random.sample's
//     pool/set switch at setsize = 21 + 4**ceil(log(3k, 4)) (k > 5).
// Python's own loop costs ~43 ms per level at config 3; this is
// microseconds.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "../ams_host.h"

namespace ams {

// ---------------------------------------------------------------- BLAKE2b
namespace {
const uint64_t kIV[8] = {
    0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
    0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
    0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};
const uint8_t kSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

inline uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

void compress(uint64_t h[8], const uint8_t block[128], uint64_t t, bool last) {
  uint64_t m[16], v[16];
  for (int i = 0; i < 16; ++i) {
    uint64_t w = 0;
    for (int b = 7; b >= 0; --b) w = (w << 8) | block[8 * i + b];
    m[i] = w;
  }
  for (int i = 0; i < 8; ++i) { v[i] = h[i]; v[i + 8] = kIV[i]; }
  v[12] ^= t;  // messages here are far below 2^64 bytes
  if (last) v[14] = ~v[14];
  auto G = [&](int a, int b, int c, int d, uint64_t x, uint64_t y) {
    v[a] = v[a] + v[b] + x; v[d] = rotr(v[d] ^ v[a], 32);
    v[c] = v[c] + v[d];     v[b] = rotr(v[b] ^ v[c], 24);
    v[a] = v[a] + v[b] + y; v[d] = rotr(v[d] ^ v[a], 16);
    v[c] = v[c] + v[d];     v[b] = rotr(v[b] ^ v[c], 63);
  };
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = kSigma[r];
    G(0, 4, 8, 12, m[s[0]], m[s[1]]);
    G(1, 5, 9, 13, m[s[2]], m[s[3]]);
    G(2, 6, 10, 14, m[s[4]], m[s[5]]);
    G(3, 7, 11, 15, m[s[6]], m[s[7]]);
    G(0, 5, 10, 15, m[s[8]], m[s[9]]);
    G(1, 6, 11, 12, m[s[10]], m[s[11]]);
    G(2, 7, 8, 13, m[s[12]], m[s[13]]);
    G(3, 4, 9, 14, m[s[14]], m[s[15]]);
  }
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}
}  // namespace

void blake2b_128(const uint8_t* msg, size_t len, uint8_t out[16]) {
  uint64_t h[8];
  for (int i = 0; i < 8; ++i) h[i] = kIV[i];
  h[0] ^= 0x01010000ULL ^ 16ULL;  // fanout=1, depth=1, no key, 16-byte digest
  uint8_t block[128];
  size_t off = 0;
  while (len - off > 128) {
    compress(h, msg + off, off + 128, false);
    off += 128;
  }
  std::memset(block, 0, sizeof block);
  std::memcpy(block, msg + off, len - off);
  compress(h, block, len, true);
  for (int i = 0; i < 16; ++i) out[i] = (uint8_t)(h[i / 8] >> (8 * (i % 8)));
}

// Seed words of random.Random(int.from_bytes(digest, "big")) — CPython
// random_seed(): 32-bit chunks of |x| from the right, keyused =
// (bits-1)//32 + 1 (1 for x == 0).
int stream_seed_words(const std::string& text, uint32_t words[4]) {
  uint8_t d[16];
  blake2b_128(reinterpret_cast<const uint8_t*>(text.data()), text.size(), d);
  for (int w = 0; w < 4; ++w) {
    const uint8_t* p = d + 12 - 4 * w;  // least significant word first
    words[w] = ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) |
               ((uint32_t)p[2] << 8) | (uint32_t)p[3];
  }
  int n = 4;
  while (n > 1 && words[n - 1] == 0) --n;
  return n;
}

// ---------------------------------------------------------------- MT19937
void Mt19937::init_genrand(uint32_t s) {
  mt[0] = s;
  for (int i = 1; i < kN; ++i)
    mt[i] = 1812433253U * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (uint32_t)i;
  index = kN;
}

// init_by_array always starts from init_genrand(19650218): computed once.
static const Mt19937& genrand_19650218() {
  static const Mt19937 base = [] {
    Mt19937 m;
    m.init_genrand(19650218U);
    return m;
  }();
  return base;
}

void Mt19937::init_by_array(const uint32_t* key, int key_length) {
  std::memcpy(mt, genrand_19650218().mt, sizeof mt);
  int i = 1, j = 0;
  for (int k = (kN > key_length ? kN : key_length); k; --k) {
    mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525U)) + key[j] + (uint32_t)j;
    ++i; ++j;
    if (i >= kN) { mt[0] = mt[kN - 1]; i = 1; }
    if (j >= key_length) j = 0;
  }
  for (int k = kN - 1; k; --k) {
    mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941U)) - (uint32_t)i;
    ++i;
    if (i >= kN) { mt[0] = mt[kN - 1]; i = 1; }
  }
  mt[0] = 0x80000000U;
  index = kN;
}

// The twist is done one word at a time, as the words are consumed: word kk
// of the new state depends on old words kk and kk + 1 and on word
// kk + kM mod kN, which is old below kN - kM and already new above — the
// same values the whole-array twist uses, in the same order.  Draws that
// use few words (most sample streams) skip the rest of the twist.
uint32_t Mt19937::next() {
  static const uint32_t mag01[2] = {0x0U, 0x9908b0dfU};
  if (index >= kN) index = 0;
  const int kk = index++;
  const int k1 = kk + 1 < kN ? kk + 1 : 0;
  const int km = kk + kM < kN ? kk + kM : kk + kM - kN;
  uint32_t y = (mt[kk] & 0x80000000U) | (mt[k1] & 0x7fffffffU);
  y = mt[km] ^ (y >> 1) ^ mag01[y & 1U];
  mt[kk] = y;
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680U;
  y ^= (y << 15) & 0xefc60000U;
  y ^= (y >> 18);
  return y;
}

// Random.getrandbits(k), 1 <= k <= 64: little-endian 32-bit words, the
// most significant one shifted down to the remaining bit count.
uint64_t Mt19937::getrandbits(int k) {
  if (k <= 32) return next() >> (32 - k);
  uint64_t lo = next();
  uint64_t hi = next() >> (64 - k);
  return lo | (hi << 32);
}

static int bit_length(uint64_t n) { return n ? 64 - __builtin_clzll(n) : 0; }

// Random._randbelow_with_getrandbits (CPython 3.12 random.py).
uint64_t Mt19937::randbelow(uint64_t n) {
  int k = bit_length(n);
  uint64_t r = getrandbits(k);
  while (r >= n) r = getrandbits(k);
  return r;
}

// sorted(Random.sample(range(n), k)).
void python_sample_sorted(Mt19937& rng, uint64_t n, uint64_t k, uint64_t* out) {
  if (k == 0) return;
  uint64_t setsize = 21;
  if (k > 5) {
    double e = std::ceil(std::log((double)(k * 3)) / std::log(4.0));
    setsize += (uint64_t)1 << (2 * (int)e);
  }
  if (n <= setsize) {
    std::vector<uint64_t> pool(n);
    for (uint64_t i = 0; i < n; ++i) pool[i] = i;
    for (uint64_t i = 0; i < k; ++i) {
      uint64_t j = rng.randbelow(n - i);
      out[i] = pool[j];
      pool[j] = pool[n - i - 1];
    }
  } else {
    // CPython keeps a set of the picks and redraws duplicates; an
    // open-addressing table (reused per thread) gives the same picks.
    thread_local std::vector<uint64_t> table;
    uint64_t cap = 16;
    while (cap < 4 * k) cap <<= 1;
    table.assign(cap, ~0ULL);
    const uint64_t mask = cap - 1;
    auto insert = [&](uint64_t v) -> bool {  // false if already present
      uint64_t h = (v * 0x9E3779B97F4A7C15ULL) >> 20;
      for (;; ++h) {
        uint64_t& e = table[h & mask];
        if (e == v) return false;
        if (e == ~0ULL) { e = v; return true; }
      }
    };
    for (uint64_t i = 0; i < k; ++i) {
      uint64_t j = rng.randbelow(n);
      while (!insert(j)) j = rng.randbelow(n);
      out[i] = j;
    }
  }
  std::sort(out, out + k);
}

}  // namespace ams

using namespace ams;

extern "C" {

int ams_stream_seed(int64_t master_seed, const char* stream_id, uint32_t out_words[4],
                    int* out_nwords) {
  if (!stream_id || !out_words) return set_error(AMS_EINVAL, "null argument");
  std::string text = std::to_string(master_seed) + "\x1f" + stream_id + "\x1f";
  int n = stream_seed_words(text, out_words);
  if (out_nwords) *out_nwords = n;
  return AMS_OK;
}

int ams_blake2b_128(const uint8_t* msg, uint64_t len, uint8_t out[16]) {
  if ((!msg && len) || !out) return set_error(AMS_EINVAL, "null argument");
  blake2b_128(msg, len, out);
  return AMS_OK;
}

int ams_sample_indices(const uint32_t* seed_words, int nwords, uint64_t n, uint64_t k,
                       uint64_t* out) {
  if (nwords < 1 || nwords > 4 || !seed_words) return set_error(AMS_EINVAL, "bad seed words");
  if (k > n) return set_error(AMS_EINVAL, "Sample larger than population or is negative");
  Mt19937 rng;
  rng.init_by_array(seed_words, nwords);
  python_sample_sorted(rng, n, k, out);
  return AMS_OK;
}

int ams_mt_getrandbits(const uint32_t* seed_words, int nwords, int k, uint64_t count,
                       uint64_t* out) {
  if (nwords < 1 || nwords > 4 || k < 1 || k > 64) return set_error(AMS_EINVAL, "bad args");
  Mt19937 rng;
  rng.init_by_array(seed_words, nwords);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.getrandbits(k);
  return AMS_OK;
}

// draw_sample (ams.py:157-175) for every group of one level, as positions.
//   Group g has members [group_first[g], group_first[g] + group_npe[g]) in
//   the PE numbering (the PE id names the stream "pe{id}"), member sizes
//   sizes[pe] and member offsets offs[pe] in the level buffer.  Its stream
//   prefix is "{stream}/L{level}-g{group_lo}/sample" (ams.py:226, 290).
//   Output per sample element: idx = offs[pe] + index (buffer position) and
//   gpos = position in the group buffer (sum of earlier members' sizes +
//   index), concatenated group by group; out_group_count[g] = drawn.
int ams_draw_sample_positions(int64_t master_seed, const char* stream, int level,
                              int ngroups, const int32_t* group_first, const int32_t* group_npe,
                              const uint64_t* targets, const uint64_t* sizes,
                              const uint64_t* offs, uint64_t capacity, uint64_t* out_idx,
                              uint64_t* out_gpos, uint64_t* out_group_count) {
  if (!stream) return set_error(AMS_EINVAL, "null stream");
  // Serial pass: every PE's quota, output slot and group position.
  struct Job {
    int pe;
    int group_lo;
    uint64_t take, out, gpos;
  };
  std::vector<Job> jobs;
  uint64_t w = 0;
  for (int g = 0; g < ngroups; ++g) {
    const int first = group_first[g], P = group_npe[g];
    uint64_t n_g = 0;
    for (int i = 0; i < P; ++i) n_g += sizes[first + i];
    if (targets[g] > n_g) {
      return set_error(AMS_EINVAL, "sample of " + std::to_string(targets[g]) +
                                       " exceeds data size " + std::to_string(n_g));
    }
    const uint64_t base = targets[g] / P, extra = targets[g] % P;
    uint64_t drawn = 0, gpos = 0;
    for (int i = 0; i < P; ++i) {
      const int pe = first + i;
      const uint64_t quota = base + ((uint64_t)i < extra ? 1 : 0);
      const uint64_t take = std::min<uint64_t>(quota, sizes[pe]);
      if (w + take > capacity) return set_error(AMS_EINVAL, "sample capacity exceeded");
      if (take) jobs.push_back({pe, first, take, w, gpos});
      w += take;
      drawn += take;
      gpos += sizes[pe];
    }
    out_group_count[g] = drawn;
  }
  // The streams are independent: draw them in parallel.
  const std::string prefix = std::to_string(master_seed) + "\x1f" + stream + "/L" +
                             std::to_string(level) + "-g";
  parallel_for((int)jobs.size(), [&](int i) {
    const Job& j = jobs[i];
    const std::string text = prefix + std::to_string(j.group_lo) + "/sample/pe" +
                             std::to_string(j.pe) + "\x1f";
    uint32_t words[4];
    const int nw = stream_seed_words(text, words);
    Mt19937 rng;
    rng.init_by_array(words, nw);
    uint64_t* idx = out_idx + j.out;
    python_sample_sorted(rng, sizes[j.pe], j.take, idx);
    for (uint64_t t = 0; t < j.take; ++t) {
      out_gpos[j.out + t] = j.gpos + idx[t];
      idx[t] += offs[j.pe];
    }
  });
  return AMS_OK;
}

}  // extern "C"

// Internal host-side declarations shared by the C-ABI translation units.
#pragma once
#include <cstdint>
#include <functional>
#include <string>

#include "../../include/ams_b200.h"

namespace ams {

// Thread-local last-error string (ams_last_error); returns `code`.
int set_error(int code, const std::string& msg);

void blake2b_128(const uint8_t* msg, size_t len, uint8_t out[16]);
int stream_seed_words(const std::string& text, uint32_t words[4]);

struct Mt19937 {
  static constexpr int kN = 624, kM = 397;
  uint32_t mt[kN];
  int index = kN + 1;
  void init_genrand(uint32_t s);
  void init_by_array(const uint32_t* key, int key_length);
  uint32_t next();
  uint64_t getrandbits(int k);
  uint64_t randbelow(uint64_t n);
};

void python_sample_sorted(Mt19937& rng, uint64_t n, uint64_t k, uint64_t* out);

// Runs f(0..count-1) on a persistent host worker pool (and the caller).
void parallel_for(int count, const std::function<void(int)>& f);

}  // namespace ams

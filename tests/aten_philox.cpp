// Independent Philox4x32-10 for pinning the oracle: ATen's header-only
// at::philox_engine (torch/include/ATen/core/PhiloxRNGEngine.h), compiled
// for the CPU at test time.  Reads "seed stream pos" triples from stdin and
// prints the four 32-bit words of block `pos` of (seed, stream).
#include <ATen/core/PhiloxRNGEngine.h>
#include <cinttypes>
#include <cstdio>

int main() {
  unsigned long long seed, stream, pos;
  while (std::scanf("%llu %llu %llu", &seed, &stream, &pos) == 3) {
    at::philox_engine eng(seed, stream, pos);
    uint32_t w0 = eng(), w1 = eng(), w2 = eng(), w3 = eng();
    std::printf("%u %u %u %u\n", w0, w1, w2, w3);
  }
  return 0;
}

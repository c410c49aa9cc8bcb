// Host build of the __host__ __device__ solver cores, for CPU-side unit tests
// only (tests/test_hostcheck.py).  Lets the CPU suite exercise the exact
// source the GPU kernels compile — P3P, the numpy-compatible sampler and the
// seeding — against the oracle without a GPU.  Not used by the package API
// (which has no CPU path) and built as a separate library.
#include <cstdint>
#include "vl_p3p.cuh"
#include "vl_rng.cuh"

using namespace vl;

extern "C" {

int vlh_p3p_solve_one(const double* f, const double* P, double* R, double* t) {
  return p3p_solve_one(f, P, R, t);
}

int vlh_quartic_roots(const double* c, double* out) { return quartic_real_pos_roots(c, out); }

// Sequential exact sampling through the same WordReader/choice3 code, plus
// the speculative path, to check they agree.  Returns words consumed.
uint64_t vlh_sample(uint64_t seed, int64_t n, int count, int64_t* out, int* n_rejections) {
  GenState g = seed_pcg64(seed);
  uint64_t pos = 0;
  int rej = 0;
  const int D = draws_per_sample(n);
  for (int i = 0; i < count; ++i) {
    WordReader rd;
    rd.init(g, pos);
    int64_t v[3];
    int used = 0;
    WordReader spec = rd;
    if (!choice3(spec, (uint32_t)n, false, v, nullptr)) ++rej;
    choice3(rd, (uint32_t)n, true, out + 3 * i, &used);
    if (used != D) ++rej;
    pos += used;
  }
  if (n_rejections) *n_rejections = rej;
  return pos;
}

void vlh_seed(uint64_t seed, uint64_t* out4) {
  GenState g = seed_pcg64(seed);
  out4[0] = (uint64_t)(g.state >> 64);
  out4[1] = (uint64_t)g.state;
  out4[2] = (uint64_t)(g.inc >> 64);
  out4[3] = (uint64_t)g.inc;
}

}  // extern "C"

/* ===========================================================================
 * fftw3.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The subset of FFTW3's complex-DFT API the reference's hot path calls
 * (nfft.cpp:379-384,409,423; kernels.cpp:296-307; detail/fftw.hpp:10-23),
 * backed by the oracle's own transform (oracle/linalg.hpp fft_nd: radix-2
 * for powers of two, direct DFT otherwise; FFTW's sign convention, no
 * normalisation), so the reference's sources compile here unchanged into
 * oracle/_ref (build_ref.sh).  FFTW3 itself is absent from this image.
 * Planner flags are accepted and ignored; plans must be cubic (n[t] equal),
 * which is every plan the reference makes ({M, M, M} / {N, N, N}).
 * =========================================================================== */
#pragma once

#include <complex>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../linalg.hpp"

typedef double fftw_complex[2];

struct fftw_plan_s {
  int rank;
  int n;
  int sign;
};
typedef fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_DESTROY_INPUT (1U << 0)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

inline fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex*, fftw_complex*, int sign, unsigned) {
  if (rank < 1 || rank > 3) return nullptr;
  for (int t = 1; t < rank; ++t)
    if (n[t] != n[0]) return nullptr;
  return new fftw_plan_s{rank, n[0], sign};
}

inline void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  size_t total = orc_linalg::ipow(static_cast<size_t>(p->n), p->rank);
  if (in != out) std::memcpy(out, in, sizeof(fftw_complex) * total);
  orc_linalg::fft_nd(reinterpret_cast<std::complex<double>*>(out), p->rank, p->n, p->sign);
}

inline void fftw_destroy_plan(fftw_plan p) { delete p; }
inline void* fftw_malloc(size_t bytes) { return std::malloc(bytes); }
inline void fftw_free(void* p) { std::free(p); }

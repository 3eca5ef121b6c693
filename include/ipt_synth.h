/*
 * ipt_synth.h — seeded synthetic inputs of BASELINE.json's five configurations.
 *
 * The random stream is the reference's xoshiro256++ seeded through splitmix64
 * (proj/include/ipt/rng.hpp:13-82, Box-Muller normal with one cached spare);
 * the draw orders are the ones SURVEY.md §8(d) fixes, so the same arrays feed
 * the device path, the CPU oracle and the reference build, and the recorded
 * anchors (e.g. Lambda_0 of config 1) reproduce. Output is host memory.
 */
#ifndef IPT_SYNTH_H
#define IPT_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Configs 1-3: d_i = i+1; Delta symmetric, zero diagonal, Delta_ij = Delta_ji =
 * eps*(2u-1) drawn over the upper triangle row-major from Rng(stream_seed(seed,0)).
 * delta: n*n row-major. */
int ipt_synth_dense_uniform(int64_t n, double eps, uint64_t seed, double* d, double* delta);

/* Config 4: d = sort(n * u_i) + i from stream 0; row i of the upper triangle from
 * stream i+1 as sigma*normal(), mirrored; zero diagonal. threads <= 0: all cores. */
int ipt_synth_dense_normal(int64_t n, double sigma, uint64_t seed, int threads, double* d,
                           double* delta);

/* Config 5 (CI-like CSR): energies 10*log1p(i) + 0.5u (stream 0) sorted; per row i,
 * `per_row` distinct partners j != i drawn with below(n) from stream 1, keys
 * min*n+max sorted and deduplicated; values sigma*normal() from stream 2 in key
 * order, mirrored. Two calls: plan (returns nnz through *nnz and an opaque handle),
 * then fill (frees the handle). rowptr: n+1, cols: nnz (sorted per row), vals: nnz. */
int ipt_synth_csr_ci_plan(int64_t n, int per_row, uint64_t seed, void** handle, int64_t* nnz);
int ipt_synth_csr_ci_fill(void* handle, double sigma, double* d, int64_t* rowptr, int32_t* cols,
                          double* vals);

/* Raw draws of the generator, for pinning against the reference's Rng.
 * kind 0 = next(), 1 = uniform(), 2 = normal(), 3 = below(bound). */
void ipt_synth_rng_draws(uint64_t seed, uint64_t stream, int use_stream, int kind, uint64_t bound,
                         int64_t count, void* out);

#ifdef __cplusplus
}
#endif

#endif /* IPT_SYNTH_H */

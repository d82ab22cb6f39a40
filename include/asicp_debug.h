/*
 * asicp_debug.h — component entry points used by the parity tests.
 *
 * Not part of the drop-in boundary.  They expose single building blocks of
 * the solver so tests can pin them individually against the reference:
 *   asicp_dbg_exp_host / _device: the glibc-exact exp of the SVGD kernel
 *     (rbf_kernel, optim.cpp:120-125) on the host and on the GPU.
 */
#ifndef ASICP_DEBUG_H_
#define ASICP_DEBUG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

void asicp_dbg_exp_host(const double* x, double* y, int64_t n);
/* Returns 0 on success, ASICP_DEVICE_ERROR on a CUDA failure. */
int asicp_dbg_exp_device(const double* x, double* y, int64_t n);

/* FP32 FFMA throughput microbenchmark on the current device (the roofline
 * denominator of the NN filter): every SM runs independent FFMA chains for
 * `iters` iterations; returns achieved TFLOP/s (2 FLOP per FFMA), timed with
 * CUDA events, or a negative value on failure. */
double asicp_dbg_ffma_tflops(int iters);
double asicp_dbg_dfma_tflops(int iters);  /* FP64 DFMA throughput (TFLOP/s) */

/* Raw NN counters of the last asicp_run: [0] windows decided in FP64, [1] full
 * FP64 rescans, [2] queries, [3] canonical-order ties, [4] pairs, [5..7] rescans
 * per match kind (forward, reverse, final), [8..11] rescan reasons (mode,
 * top-3 overflow, window > list, merge overflow), [16 + k] full rescans in
 * iteration k (k_max = final ranking).  `out` holds 256 entries. */
struct asicp_ctx;
int asicp_dbg_raw_stats(struct asicp_ctx* ctx, uint64_t* out);

/* Per-iteration NN work of the last asicp_run: for k = 0..k_max (k_max = the
 * final ranking) out[4k + 0/1] = forward/reverse (query, candidate) pairs,
 * out[4k + 2/3] = forward/reverse queries.  Copies min(n, 4 (k_max + 1))
 * entries; returns 4 (k_max + 1), or -1 (no prepared problem / in flight). */
int64_t asicp_dbg_iter_stats(struct asicp_ctx* ctx, uint64_t* out, int64_t n);

/* The device minibatch sampler (mt19937_64 + Lemire + partial Fisher-Yates,
 * spatial_index.cpp:111-123) on one stream seeded with `seed`: `calls`
 * consecutive draws of ms[c] indices from [0, n), written back to back.
 * parallel != 0 selects the parallel (sort + pointer-jumping) kernel where
 * it applies, 0 the serial swap kernel. */
int asicp_dbg_minibatch(uint64_t seed, int64_t n, const int64_t* ms, int64_t calls, int32_t parallel, int32_t* out);

#ifdef __cplusplus
}
#endif

#endif /* ASICP_DEBUG_H_ */

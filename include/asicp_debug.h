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

#ifdef __cplusplus
}
#endif

#endif /* ASICP_DEBUG_H_ */

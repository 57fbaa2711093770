/*
 * protea_selftest.h — hardware self-test entry of libprotea.so (not part of the
 * round API).  Runs the library's tcgen05/TMEM GEMM core on dense bf16
 * operands so that the tensor-core descriptor encodings can be checked in
 * isolation against a plain matmul (tests/test_gpu_tc.py).
 */
#ifndef PROTEA_SELFTEST_H
#define PROTEA_SELFTEST_H
#include "protea.h"
#ifdef __cplusplus
extern "C" {
#endif

/* D[M][N] (fp32, device) = sum_k A[m][k] B[n][k] with A, B bf16 device arrays:
 * mn_major == 0: A is [M][K], B is [N][K] (K-major operands);
 * mn_major == 1: A is [K][M], B is [K][N] (MN-major operands).
 * M % 128 == 0, 0 < N <= 64, K % 64 == 0.  Synchronises the device.
 * Errors: INVALID, CUDA. */
protea_status protea_selftest_gemm(const void* A, const void* B, float* D, int32_t M, int32_t N, int32_t K,
                                   int32_t mn_major);

#ifdef __cplusplus
}
#endif
#endif

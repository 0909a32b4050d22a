/*
 * fl_debug.h — test-only introspection of libfl_b200.so (not needed by users).
 *
 * fl_debug_read copies one of the CNN's per-slot activation buffers of the LAST
 * SGD wave run by fl_train_clients to host memory, so kernel-level tests can compare
 * the tensor-core path (math = 0) with the FP32 SIMT path (math = 1) layer by layer.
 * Buffers are slot-major NHWC, slot (a, r) = a·B + r, a = execution index of an
 * active client:
 *   "p1" f32 [S][H1][W1][C1]  "am1" u8 same   "p2" f32 [S][H2][W2][C2]  "am2" u8 same
 *   "h" / "dh" f32 [S][HID]   "dp2" f32 [S][F] "dY2" f32 [S][H1][W1][C2]
 *   "dp1" f32 [S][H1][W1][C1] "dY1" f32 [S][H0][W0][C1]
 * "sig" (any model): the ctx's peer signal words uint64 [(8 + 1)·T] (ready[8][T], done[T]),
 * copied without waiting for the ctx stream (to inspect a peer aggregation in flight).
 * bytes is the caller's buffer size; copies min(bytes, buffer size).  Synchronous.
 * FL_ERR_INVALID for an unknown name or a non-CNN context.
 */
#ifndef FL_B200_DEBUG_H
#define FL_B200_DEBUG_H
#include <stdint.h>
#include "fl.h"
#ifdef __cplusplus
extern "C" {
#endif
fl_status fl_debug_read(fl_ctx* ctx, const char* name, void* host, int64_t bytes);
#ifdef __cplusplus
}
#endif
#endif

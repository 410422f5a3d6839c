// tr_internal.h -- shared helpers of libtetray_b200 (not part of the C ABI).
#pragma once
#include <cstdint>

// Record an error message for tr_last_error() and return code.
int tr_fail(int code, const char *msg);
// K:74-90 on the host (used by the TF-metadata restatement).
void tr_tf_sample_host(const double *T, int64_t n, double lo, double hi, double v, double *rgba);
// Walk table (TrPLeaf.walk) of a generator cube of the given parity (mesh.py:151-163).
extern "C" void tr_walk_table_cube(int parity, uint32_t walk[8]);

// rubs_internal.h -- helpers shared by the translation units of librubs_b200
// (not part of the C ABI).
#pragma once

#include <cstdint>
#include <string>

struct rubs_lut;

namespace rubs_internal {

// Thread-local host state (scratch buffers, streams, events) is kept per
// CUDA device: a single-process caller that alternates devices keeps each
// device's buffers and streams instead of dropping (leaking) them, and no
// kernel is handed another device's memory.  Index = the current device,
// checked against the bound by each translation unit's ensure function.
constexpr int kMaxDevices = 16;

// Record the thread's last error message (rubs_b200_last_error) and return
// `code`.
int set_error(int code, const std::string &msg);

// Launch accounting shared by the translation units: count `n` kernel
// launches (rubs_b200_launch_count), and bracket the primary filter launch
// of a pass with CUDA events when profiling is on (rubs_b200_kernel_time,
// kind 0 = primary filter kernel); timer_collect() after the stream sync.
void count_launches(int n);
void *timed_begin(int kind, void *stream);
void timed_end(void *token);
void timer_collect();

// Largest elongation of a LUT's rho grid.
double lut_rho_max(const rubs_lut *lut);

// One filter pass of 1-3 channels (same geometry / dtype / strides) that
// share the per-pixel kernel: a uniform scale-vector, or LUT parameters.
// Results equal the single-channel calls bit for bit.
int filter_uniform_multi(const double *const *f, int nch, int64_t H, int64_t W, int64_t ld,
                         const double a[4], double *const *out, int64_t ld_out, void *stream);
int filter_params_multi(const void *const *f, int f_dtype, int nch, int64_t H, int64_t W,
                        int64_t ld, const void *size, const void *elong, const void *orient,
                        int p_dtype, int64_t ld_p, const rubs_lut *lut, double *const *out,
                        int64_t ld_out, void *stream);

}  // namespace rubs_internal

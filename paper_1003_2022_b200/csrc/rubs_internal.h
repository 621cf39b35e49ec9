// rubs_internal.h -- helpers shared by the translation units of librubs_b200
// (not part of the C ABI).
#pragma once

#include <string>

struct rubs_lut;

namespace rubs_internal {

// Record the thread's last error message (rubs_b200_last_error) and return
// `code`.
int set_error(int code, const std::string &msg);

// Largest elongation of a LUT's rho grid.
double lut_rho_max(const rubs_lut *lut);

}  // namespace rubs_internal

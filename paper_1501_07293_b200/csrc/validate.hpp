// validate.hpp — device self-check suite behind mmb_validate (validate.cu).
#pragma once

#include <string>

namespace mmb {

// Runs every check; returns the report (one "PASS|FAIL  name: detail" line per check, then
// "all checks passed" or "VALIDATION FAILED", like render_report, proj/src/validate.cpp:192-198).
std::string run_device_validation(bool& all_passed);

} // namespace mmb

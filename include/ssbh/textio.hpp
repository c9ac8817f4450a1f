// ssbh/textio.hpp — declaration of the reference's report formatter
// (proj/include/ssbh/textio.hpp; defined in its proj/src/pipeline.cpp, host-side).
#pragma once

#include <string>

namespace ssbh {

/// Locale-independent shortest round-trip decimal form of a double.
std::string double_to_string(double v);

}  // namespace ssbh

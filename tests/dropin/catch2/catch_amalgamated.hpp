// Catch2 stand-in for the reference's unit suites (proj/tests/*.cpp): they use
// only TEST_CASE / REQUIRE / REQUIRE_FALSE / REQUIRE_NOTHROW /
// REQUIRE_THROWS_AS / INFO.  Catch2 itself is not in this image.
#pragma once
#include <sstream>

#include "../../cpp/minicatch.hpp"

#define INFO(msg)                 \
  do {                            \
    std::ostringstream mc_info_;  \
    mc_info_ << msg;              \
  } while (0)

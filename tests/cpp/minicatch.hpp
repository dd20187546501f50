// minicatch.hpp -- the subset of Catch2's interface the reference's tests use
// (TEST_CASE / REQUIRE / REQUIRE_FALSE / REQUIRE_THROWS_AS / REQUIRE_NOTHROW),
// so these tests read like proj/tests/*.cpp.  Run: <binary> [tag-substring].
#pragma once
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace minicatch {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
struct Failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
inline int run(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : "";
  int failed = 0, ran = 0;
  for (auto& c : cases()) {
    if (*filter && !std::strstr(c.name, filter)) continue;
    ++ran;
    try {
      c.fn();
      std::printf("PASS %s\n", c.name);
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAIL %s: %s\n", c.name, e.what());
    }
  }
  std::printf("%d/%d passed\n", ran - failed, ran);
  return failed ? 1 : 0;
}
}  // namespace minicatch

#define MC_CAT2(a, b) a##b
#define MC_CAT(a, b) MC_CAT2(a, b)
#define TEST_CASE(name)                                                          \
  static void MC_CAT(mc_test_, __LINE__)();                                      \
  static minicatch::Reg MC_CAT(mc_reg_, __LINE__)(name, MC_CAT(mc_test_, __LINE__)); \
  static void MC_CAT(mc_test_, __LINE__)()
#define MC_STR2(x) #x
#define MC_STR(x) MC_STR2(x)
#define REQUIRE(...)                                                                                   \
  do {                                                                                                 \
    if (!(__VA_ARGS__)) throw minicatch::Failure(__FILE__ ":" MC_STR(__LINE__) ": REQUIRE(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define REQUIRE_THROWS_AS(expr, type)                                                          \
  do {                                                                                         \
    bool mc_ok = false;                                                                        \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const type&) {                                                                    \
      mc_ok = true;                                                                            \
    }                                                                                          \
    if (!mc_ok) throw minicatch::Failure(__FILE__ ":" MC_STR(__LINE__) ": no " #type " from " #expr); \
  } while (0)
#define REQUIRE_NOTHROW(...) (void)(__VA_ARGS__)

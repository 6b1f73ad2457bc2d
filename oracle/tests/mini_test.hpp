// Tiny doctest-shaped harness (doctest itself is absent from the image):
// TEST_CASE / CHECK / REQUIRE / CHECK_THROWS_AS / Approx.  Prints one line
// per failure and a summary; exit code = number of failed cases.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace mt {
struct Case { const char* name; std::function<void()> fn; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
struct Reg { Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); } };
struct RequireFail {};

struct Approx {
  double v, eps = 1e-12 * 100;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  friend bool operator==(double a, const Approx& b) {
    return std::abs(a - b.v) <= b.eps * (1.0 + std::max(std::abs(a), std::abs(b.v)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
};

inline int run_all(const char* filter = nullptr) {
  int failed_cases = 0, ran = 0;
  for (auto& c : registry()) {
    if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
    const int before = failures();
    ++ran;
    try {
      c.fn();
    } catch (RequireFail&) {
    } catch (std::exception& e) {
      std::printf("  EXCEPTION in [%s]: %s\n", c.name, e.what());
      ++failures();
    }
    if (failures() != before) {
      ++failed_cases;
      std::printf("FAILED: %s\n", c.name);
    } else {
      std::printf("ok: %s\n", c.name);
    }
  }
  std::printf("== %d cases, %d failed, %d checks\n", ran, failed_cases, checks());
  return failed_cases;
}
}  // namespace mt

#define MT_CAT2(a, b) a##b
#define MT_CAT(a, b) MT_CAT2(a, b)
#define TEST_CASE(name)                                                       \
  static void MT_CAT(mt_fn_, __LINE__)();                                     \
  static mt::Reg MT_CAT(mt_reg_, __LINE__)(name, &MT_CAT(mt_fn_, __LINE__)); \
  static void MT_CAT(mt_fn_, __LINE__)()
#define CHECK(cond)                                                             \
  do {                                                                          \
    ++mt::checks();                                                             \
    if (!(cond)) {                                                              \
      ++mt::failures();                                                         \
      std::printf("  %s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #cond);     \
    }                                                                           \
  } while (0)
#define REQUIRE(cond)                                                           \
  do {                                                                          \
    ++mt::checks();                                                             \
    if (!(cond)) {                                                              \
      ++mt::failures();                                                         \
      std::printf("  %s:%d REQUIRE(%s) failed\n", __FILE__, __LINE__, #cond);   \
      throw mt::RequireFail{};                                                  \
    }                                                                           \
  } while (0)
#define CHECK_THROWS_AS(expr, Type)                                             \
  do {                                                                          \
    ++mt::checks();                                                             \
    bool mt_ok = false;                                                         \
    try { (void)(expr); } catch (const Type&) { mt_ok = true; } catch (...) {}  \
    if (!mt_ok) {                                                               \
      ++mt::failures();                                                         \
      std::printf("  %s:%d CHECK_THROWS_AS(%s, %s) failed\n", __FILE__, __LINE__, #expr, #Type); \
    }                                                                           \
  } while (0)
#define MT_MAIN \
  int main(int argc, char** argv) { return mt::run_all(argc > 1 ? argv[1] : nullptr); }

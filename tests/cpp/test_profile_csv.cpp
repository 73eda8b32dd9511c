// CPU test: profile samples round-trip through the CSV ingest SPEC.md:592
// promises (optimizer.hpp read/write_profile_csv) and fit identically.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <sstream>

#include "moeplan/optimizer.hpp"

using namespace moeplan;

TEST_CASE("profile CSV round trip preserves samples and the fitted model") {
  std::vector<ProfileSample> s;
  for (int i = 1; i <= 5; ++i) {
    s.push_back({EventKind::H2D_EXPERTS, 2.8186e9 * i / 5.0, 1e-3 + 0.0180 * i / 5.0 + 1e-9 * i});
    s.push_back({EventKind::CPU_ATTN, 3.2e5 * i, 2e-5 + 1e-10 * 3.2e5 * i});
    s.push_back({EventKind::DRAFT_GPU_STEP, 32.0 * 1024 * i, 1e-4 * i / 3.0});
  }
  std::ostringstream out;
  write_profile_csv(s, out);
  std::istringstream in("# measured on B200\n" + out.str() + "\n");
  const std::vector<ProfileSample> r = read_profile_csv(in);
  REQUIRE(r.size() == s.size());
  for (size_t i = 0; i < s.size(); ++i) {
    CHECK(r[i].kind == s[i].kind);
    CHECK(r[i].driving == s[i].driving);  // max_digits10: exact round trip
    CHECK(r[i].seconds == s[i].seconds);
  }
  const LatencyModel a = fit_latency_models(s), b = fit_latency_models(r);
  CHECK(a.size() == b.size());
  for (const auto& kv : a) {
    CHECK(b.at(kv.first).slope == kv.second.slope);
    CHECK(b.at(kv.first).intercept == kv.second.intercept);
  }
}

TEST_CASE("profile CSV errors") {
  std::istringstream bad_header("kind,x,y\nGPU_MOE,1,2\n");
  CHECK_THROWS_AS(read_profile_csv(bad_header), std::invalid_argument);
  std::istringstream bad_kind("kind,driving,seconds\nNOT_A_KIND,1,2\n");
  CHECK_THROWS_AS(read_profile_csv(bad_kind), std::invalid_argument);
  std::istringstream bad_num("kind,driving,seconds\nGPU_MOE,1x,2\n");
  CHECK_THROWS_AS(read_profile_csv(bad_num), std::invalid_argument);
  std::istringstream empty("");
  CHECK_THROWS_AS(read_profile_csv(empty), std::invalid_argument);
}

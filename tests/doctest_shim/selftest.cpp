// Self-test of the doctest shim: nested SUBCASE re-entry and failure detection.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
#include <cstdio>
static int leaves = 0, top = 0;
TEST_CASE("nested") {
  ++top;
  SUBCASE("a") { SUBCASE("a1") { ++leaves; } SUBCASE("a2") { ++leaves; } }
  SUBCASE("b") { ++leaves; }
}
TEST_CASE("report") { std::printf("top=%d leaves=%d\n", top, leaves); CHECK(top == 3); CHECK(leaves == 3); }
TEST_CASE("fails") { CHECK(1 == 2); REQUIRE(false); CHECK(true); }
TEST_CASE("throws") { CHECK_THROWS_AS(throw 1, int); CHECK_THROWS_AS((void)0, int); }

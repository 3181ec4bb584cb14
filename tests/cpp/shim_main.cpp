// Entry point for the C++ suites built against the drop-in headers (tests/cpp/Makefile).
#include <catch2/catch_amalgamated.hpp>

int main(int argc, char** argv) { return shim::run_all(argc, argv); }

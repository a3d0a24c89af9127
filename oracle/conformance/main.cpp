// Entry point of the conformance binaries (oracle/conformance/Makefile).
#include <gtest/gtest.h>

int main(int argc, char** argv) { return ::testing::run_all(argc, argv); }

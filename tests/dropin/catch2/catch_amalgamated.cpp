// main() for the reference suites built against the drop-in headers
// (proj/tests/catch_main.cpp includes this file).
#include "catch_amalgamated.hpp"

int main(int argc, char** argv) { return minicatch::run(argc, argv); }

// Runner entry point for the Catch2 shim.
#include <catch2/catch_amalgamated.hpp>

int main() { return Catch::shim::run_all(); }

// main() of the Catch2-compatible harness (catch_amalgamated.hpp): runs every
// registered TEST_CASE, or those whose name contains argv[1].
#include "catch_amalgamated.hpp"

int main(int argc, char** argv) { return Catch::run_all(argc > 1 ? argv[1] : nullptr); }

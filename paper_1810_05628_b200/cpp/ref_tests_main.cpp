// ref_tests_main.cpp — runner for the reference's UNMODIFIED unit tests
// (/root/reference/proj/tests/test_objectives.cpp, test_solvers.cpp,
// test_multigrid.cpp) compiled against the B200 drop-in headers
// (cpp/include/ptycho) and the doctest shim; every objective evaluation,
// FFT, transfer and GPU-resident solver runs through libptg on the B200.
#include "doctest.h"

int main() { return doctest::run_all(); }

// ptycho_b200.hpp — one-include entry to the C++ drop-in for the reference's
// public hot-path API (/root/reference/proj/include/ptycho/*.hpp): the headers
// under cpp/include/ptycho keep the reference's names, namespace (ptycho),
// types and error behaviour, over the libptg C-ABI (include/ptg.h).  Existing
// code compiles unchanged with -I cpp/include (instead of the reference's
// include directory) and links libptg.so.  `ptycho_b200` aliases the namespace.
#pragma once

#include "ptycho/errors.hpp"
#include "ptycho/field.hpp"
#include "ptycho/forward.hpp"
#include "ptycho/kernels.hpp"
#include "ptycho/multigrid.hpp"
#include "ptycho/objectives.hpp"
#include "ptycho/rng.hpp"
#include "ptycho/solvers.hpp"

namespace ptycho_b200 = ptycho;

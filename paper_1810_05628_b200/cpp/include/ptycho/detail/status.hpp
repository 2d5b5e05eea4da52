// detail/status.hpp — libptg status codes -> the reference's exception types.
#pragma once

#include <string>

#include "../errors.hpp"
#include "ptg.h"

namespace ptycho::detail {

inline void check(int rc) {
    if (rc == PTG_OK) return;
    const std::string m = ptg_last_error();
    switch (rc) {
        case PTG_ERR_GEOMETRY: throw GeometryError(m);
        case PTG_ERR_DOMAIN: throw DomainError(m);
        case PTG_ERR_METRIC: throw MetricError(m);
        case PTG_ERR_CONFIG: throw ConfigError(m);
        case PTG_ERR_IO: throw IoError(m);
        case PTG_ERR_NUMERIC: throw NumericError(m);
        case PTG_ERR_CUDA: throw CudaError(m);
        default: throw Error(m);
    }
}

inline const double* dp(const void* p) { return static_cast<const double*>(p); }
inline double* dp(void* p) { return static_cast<double*>(p); }

}  // namespace ptycho::detail

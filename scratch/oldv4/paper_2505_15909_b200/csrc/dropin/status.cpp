// status.cpp -- maps C-ABI status codes onto the reference exception classes.
#include "rtnq/error.hpp"
#include "rtnq_capi.h"

namespace rtnq {

void throw_status(int status, const std::string& msg) {
    switch (status) {
        case RTNQ_E_INVALID_INPUT: throw InvalidInputError(msg);
        case RTNQ_E_SHAPE: throw ShapeError(msg);
        case RTNQ_E_CORRUPT: throw CorruptDataError(msg);
        case RTNQ_E_PLAN: throw PlanError(msg);
        case RTNQ_E_IO: throw IoError(msg);
        case RTNQ_E_CUDA:
        case RTNQ_E_UNSUPPORTED: throw DeviceError(msg);
        default: throw Error(msg);
    }
}

}  // namespace rtnq

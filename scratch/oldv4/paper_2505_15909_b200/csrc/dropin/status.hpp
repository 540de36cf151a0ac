// status.hpp -- C-ABI status -> rtnq exception, shared by the drop-in sources.
#pragma once

#include <string>

#include "rtnq/error.hpp"
#include "rtnq_capi.h"

namespace rtnq::detail {

inline void check(rtnq_status st) {
    if (st != RTNQ_OK) throw_status(st, rtnq_last_error());
}

inline rtnq_layout to_c(const LayoutTag& t) {
    return rtnq_layout{static_cast<int32_t>(t.kind), t.tile_rows, t.tile_cols};
}

}  // namespace rtnq::detail

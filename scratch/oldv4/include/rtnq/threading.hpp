// rtnq/threading.hpp -- worker-count API (drop-in for proj/core/include/rtnq/threading.hpp).
// On the B200 the CUDA grid does the parallel work; the worker count is kept for
// source compatibility and only affects parallel_for, a host utility.  Results
// of every rtnq function are independent of it, as in the reference.
#pragma once

#include <cstdint>
#include <functional>

namespace rtnq {

void set_threads(int n);
int threads();
void parallel_for(std::int64_t n, std::int64_t min_items_per_worker,
                  const std::function<void(std::int64_t, std::int64_t)>& fn);

}  // namespace rtnq

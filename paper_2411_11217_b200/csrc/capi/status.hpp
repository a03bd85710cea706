// Exception -> status-code translation for the C ABI.  No exception crosses
// the extern "C" boundary; the message is kept thread-local
// and returned by mlt_last_error().
#pragma once

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "mlt.h"

namespace mlt {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct BudgetError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_error(const char* msg, int code = MLT_ERR_INTERNAL);
const char* last_error();
int last_status();

}  // namespace mlt

// Every typed error the planner, scheduler and runtime can raise, mapped to
// its status.  Template so each includer sees its own namespace's types.
#define MLT_GUARD_BODY(NS)                                                           \
    try {                                                                            \
        return f();                                                                  \
    } catch (const NS::InfeasiblePolicyError& e) {                                   \
        mlt::set_error(e.what(), MLT_ERR_INFEASIBLE);                                                    \
        return MLT_ERR_INFEASIBLE;                                                   \
    } catch (const NS::NoFeasiblePolicyError& e) {                                   \
        mlt::set_error(e.what(), MLT_ERR_NO_FEASIBLE);                               \
        return MLT_ERR_NO_FEASIBLE;                                                  \
    } catch (const NS::InvalidBatchParametersError& e) {                             \
        mlt::set_error(e.what(), MLT_ERR_INVALID);                                   \
        return MLT_ERR_INVALID;                                                      \
    } catch (const NS::sim::UnsupportedCombinationError& e) {                        \
        mlt::set_error(e.what(), MLT_ERR_UNSUPPORTED);                                                    \
        return MLT_ERR_UNSUPPORTED;                                                  \
    } catch (const NS::sim::CycleDetectedError& e) {                                 \
        mlt::set_error(e.what(), MLT_ERR_CYCLE);                                                    \
        return MLT_ERR_CYCLE;                                                        \
    } catch (const NS::sim::EmptyTimelineError& e) {                                 \
        mlt::set_error(e.what(), MLT_ERR_EMPTY);                                                    \
        return MLT_ERR_EMPTY;                                                        \
    } catch (const mlt::CudaError& e) {                                              \
        mlt::set_error(e.what(), MLT_ERR_CUDA);                                                    \
        return MLT_ERR_CUDA;                                                         \
    } catch (const mlt::BudgetError& e) {                                            \
        mlt::set_error(e.what(), MLT_ERR_BUDGET);                                                    \
        return MLT_ERR_BUDGET;                                                       \
    } catch (const std::invalid_argument& e) {                                       \
        mlt::set_error(e.what(), MLT_ERR_INVALID);                                                    \
        return MLT_ERR_INVALID;                                                      \
    } catch (const std::exception& e) {                                              \
        mlt::set_error(e.what(), MLT_ERR_INTERNAL);                                                    \
        return MLT_ERR_INTERNAL;                                                     \
    } catch (...) {                                                                  \
        mlt::set_error("unknown exception", MLT_ERR_INTERNAL);                                         \
        return MLT_ERR_INTERNAL;                                                     \
    }

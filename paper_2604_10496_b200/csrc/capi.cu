// Error state, launch counter and version of the cq_b200 C ABI.
#include "common.cuh"

#include <cstdlib>

namespace cq {
static thread_local std::string t_error;
std::atomic<int64_t> g_launches{0};
void set_error(const std::string &msg) { t_error = msg; }
bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("CQ_PDL");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}
}  // namespace cq

extern "C" const char *cq_last_error(void) { return cq::t_error.c_str(); }
extern "C" int cq_abi_version(void) { return 6; }
extern "C" int64_t cq_launch_count(void) { return cq::g_launches.load(); }

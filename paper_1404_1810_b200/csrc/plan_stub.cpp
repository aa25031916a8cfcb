// plan_stub.cpp -- error sink for the host-only plan library
// (build/libamqft_plan.so, used by codegen/gen_small.py at build time).
#include <string>

namespace amqft_b200 {
void set_last_error(const std::string&) {}
}  // namespace amqft_b200

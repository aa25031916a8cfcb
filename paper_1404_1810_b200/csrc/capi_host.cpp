// capi_host.cpp -- host-only C ABI entry points (no CUDA calls).
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../include/amqft_b200.h"
#include "plan.hpp"

using namespace amqft_b200;

namespace amqft_b200 {
void set_last_error(const std::string& m);
}

extern "C" amqft_status amqft_schedule_dump(int variant, int function, size_t n,
                                            size_t capacity_cells, void* records,
                                            size_t cap, size_t* count, uint32_t* stages,
                                            size_t cap2, size_t* nstages, uint64_t* ops3) {
  try {
    const Compiled c = compile(variant, function, n, capacity_cells);
    if (!c.single) {
      set_last_error("request exceeds the single-CTA capacity");
      return AMQFT_EINVAL;
    }
    const SubProgram& sp = c.progs[0];
    if (count) *count = sp.eis.size();
    if (records) std::memcpy(records, sp.eis.data(), std::min(cap, sp.eis.size()) * sizeof(EI));
    if (nstages) *nstages = sp.stages.size();
    if (stages)
      for (size_t s = 0; s < std::min(cap2, sp.stages.size()); ++s) {
        stages[2 * s] = sp.stages[s].ei_begin;
        stages[2 * s + 1] = sp.stages[s].ei_end;
      }
    if (ops3) {
      ops3[0] = c.ops.adds;
      ops3[1] = c.ops.muls;
      ops3[2] = c.ops.bt;
    }
    return AMQFT_OK;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return AMQFT_EINVAL;
  }
}

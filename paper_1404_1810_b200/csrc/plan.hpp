// plan.hpp -- host-side plan compiler for the AM-QFT recursion.
//
// Replaces the reference's per-call plan + interpreter
// (build_plan, src/variants.cpp:173-234; Executor::run, variants.cpp:313-351)
// with a one-time compilation of (variant, function, N) into a flat list of
// "elaboration instances" (EIs).  Every node of the recursion owns a
// contiguous cell range of a per-transform arena; an EI is one elaboration
// phase of one node (a split, a merge, an AM conversion, a base case) and
// maps cells of that range to cells of the same range.  EIs of one stage
// touch disjoint ranges and run in parallel; halvings are pure
// reinterpretations (elaborations.cpp:212-223) and cost nothing.
//
// Each EI performs exactly the reference's operations on the reference's
// operands in the reference's association (see the per-op comments in
// kernels_generic.cu), so an fp64 evaluation without FMA contraction is
// bitwise equal to amqft::execute.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace amqft_b200 {

// FunctionId order of the reference (include/amqft/variants.hpp:55-66).
enum Fn : int {
  kCdft = 0, kRdft, kDct, kDst, kDctOddTime, kDstOddTime, kDctOddHarm,
  kDstOddHarm, kDctOddOdd, kDstOddOdd, kNumFn
};

// EI opcodes.  Positions are relative to EI::off; `lens` is 0 for the cosine
// lens and 1 for the sine lens of the mother.
enum Op : uint8_t {
  OP_SC_F = 1,    // SplitComplex fwd: deinterleave 2n -> n + n  (elab.cpp:147-157)
  OP_SC_B,        // SplitComplex bwd: combine packed spectra   (elab.cpp:162-183)
  OP_SR_F,        // SplitReal fwd                               (elab.cpp:185-197)
  OP_SR_B,        // SplitReal bwd (copies)                      (elab.cpp:199-208)
  OP_GATHER,      // SplitTimeParity fwd (copies)                (elab.cpp:281-297)
  OP_SCATTER,     // SplitHarmonicParity bwd (copies)            (elab.cpp:261-277)
  OP_SH_F_DCT,    // SplitHarmonicParity fwd, DctFull mother     (elab.cpp:229-257)
  OP_SH_F_DST,    // SplitHarmonicParity fwd, DstFull mother
  OP_SH_F_ODD,    // SplitHarmonicParity fwd, odd-time mother
  OP_ST_B_DCT,    // SplitTimeParity bwd, DctFull mother         (elab.cpp:304-332)
  OP_ST_B_DST,    // SplitTimeParity bwd, DstFull mother
  OP_ST_B_ODD,    // SplitTimeParity bwd, odd-harmonic mother
  OP_AM_F,        // am_forward  M1..M8                          (elab.cpp:350-449)
  OP_AM_B,        // am_backward M1..M8                          (elab.cpp:451-527)
  OP_BASE_CDFT2,  // Executor::base_case Cdft n=2                (variants.cpp:359-364)
  OP_BASE_PAIR2,  // base_case Rdft/Dct n=2                      (variants.cpp:365-372)
  OP_BASE_OO8,    // base_case Dct/DstOddOdd n=8                 (variants.cpp:388-391)
  OP_CHAIN_F,     // serial M3/M7 forward recurrence (1 item)
  OP_CHAIN_B,     // serial M1/M5 backward recurrence (1 item)
};

// flags bits (global multi-pass path): source / destination buffer.
enum : uint8_t {
  FL_SRC_B = 1,   // read the mother (fwd) or both children (bwd) from buffer B
  FL_DST_B = 2,   // write into buffer B
  FL_DESC = 4,    // chain direction: descending positions
  FL_ADD = 8,     // chain sign: add (else subtract)
};

struct EI {
  uint8_t op;
  uint8_t lens;   // 0 cosine, 1 sine (mother's lens)
  uint8_t flags;
  uint8_t am;     // AM conversion number 1..8 (OP_AM_*), else 0
  uint32_t n;     // periodization of the mother
  uint32_t off;   // arena position of the node's range
  uint32_t aux;   // op-dependent: cells of child 0 (gather/scatter), q (chains/AM)
};
static_assert(sizeof(EI) == 16, "EI must stay 16 bytes");

struct Stage {
  uint32_t ei_begin, ei_end;  // [begin, end) into the EI array
  uint32_t items;             // total work items
};

// A stage program for one subtree root (function f at periodization n),
// executed by one CTA in shared memory.  Offsets are relative to the root.
struct SubProgram {
  int fn = 0;
  size_t n = 0;
  size_t cells = 0;
  std::vector<Stage> stages;   // EI ranges index `eis`
  std::vector<EI> eis;
  std::vector<uint32_t> prefix;  // per EI: exclusive item prefix within stage
  uint32_t max_items = 0;        // max items over stages
  uint32_t has_chain = 0;
};

// A subtree job of the multi-pass path: run subprogram `prog` on the
// arena range [off, off + cells) of every row, reading buffer `src` and
// writing buffer `dst` (0 = A, 1 = B).
struct Job {
  uint32_t prog;
  uint32_t off;
  uint8_t src, dst;
};

struct OpCount {
  uint64_t adds = 0, muls = 0, bt = 0;
};

// The compiled plan of one (variant, function, N).
struct Compiled {
  int variant = 0;
  int fn = 0;
  size_t n = 0;
  size_t cells = 0;          // cells of the root operand
  bool single = true;        // whole transform in one CTA (no global passes)
  std::vector<SubProgram> progs;   // progs[0] is the root when single
  // multi-pass path
  std::vector<EI> global_eis;
  std::vector<Stage> fwd_stages, bwd_stages;  // into global_eis
  std::vector<Job> jobs;
  uint8_t root_src = 0, root_dst = 0;  // arena buffer of the input / result
  OpCount ops;               // arithmetic executed by the schedule
};

// Cell count of a function's operand at periodization n
// (src/signal.cpp:254-258 via operand_type, variants.cpp:132-156).
size_t fn_cells(int fn, size_t n);
size_t fn_base(int fn);
bool fn_wired(int variant, int fn);

// Compile.  capacity_cells: largest subtree (in cells) a CTA may hold in
// shared memory; subtrees above it are split by global passes.
// Throws std::invalid_argument on a bad request.
Compiled compile(int variant, int fn, size_t n, size_t capacity_cells);

// Work items of one EI (outputs; chains count 1).
uint32_t ei_items(const EI& e);

// Arithmetic an EI performs (for schedule op accounting).
OpCount ei_ops(const EI& e);

}  // namespace amqft_b200

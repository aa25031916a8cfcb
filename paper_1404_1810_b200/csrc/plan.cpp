// plan.cpp -- AM-QFT plan compiler (see plan.hpp).
//
// The recursion wiring restated here follows build_plan
// (src/variants.cpp:173-234): Cdft -> 2 Rdft (SplitComplex); Rdft -> Dct +
// Dst (SplitReal); Dct/Dst -> reduced + odd child on the variant's major
// axis; the odd functions -> reduced + odd-odd child on the other axis; the
// odd-odd function -> AM conversion, whose halved child is exactly the
// operand of the (lens-flipped for variants 5-8) odd function at n/2, so
// Dct/DstOddOdd(n) = AM_fwd ; odd(n/2) ; AM_bwd (variants.cpp:220-231,
// 336-350 with the halvings of elaborations.cpp:212-223 as relabellings).
#include "plan.hpp"

#include <algorithm>
#include <map>
#include <stdexcept>

namespace amqft_b200 {

namespace {

[[noreturn]] void fail(const std::string& what) { throw std::invalid_argument(what); }

bool is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }
bool time_major(int v) { return v == 1 || v == 4 || v == 5 || v == 8; }

}  // namespace

size_t fn_base(int fn) {
  switch (fn) {
    case kCdft: case kRdft: case kDct: return 2;
    case kDctOddOdd: case kDstOddOdd: return 8;
    default: return 4;
  }
}

size_t fn_cells(int fn, size_t n) {
  switch (fn) {
    case kCdft: return 2 * n;
    case kRdft: return n;
    case kDct: return n / 2 + 1;
    case kDst: return n / 2 - 1;
    case kDctOddTime: case kDstOddTime: case kDctOddHarm: case kDstOddHarm: return n / 4;
    default: return n / 8;
  }
}

bool fn_wired(int v, int fn) {
  if (fn == kDctOddTime || fn == kDstOddTime) return time_major(v);
  if (fn == kDctOddHarm || fn == kDstOddHarm) return !time_major(v);
  return fn >= 0 && fn < kNumFn;
}

uint32_t ei_items(const EI& e) {
  const uint32_t n = e.n;
  switch (e.op) {
    case OP_SC_F: case OP_SC_B: return 2 * n;
    case OP_SR_F: case OP_SR_B: return n;
    case OP_GATHER: case OP_SCATTER: return n;  // n holds the mother's cell count
    case OP_SH_F_DCT: case OP_ST_B_DCT: return n / 2 + 1;
    case OP_SH_F_DST: case OP_ST_B_DST: return n / 2 - 1;
    case OP_SH_F_ODD: case OP_ST_B_ODD: return n / 4;
    case OP_AM_F: case OP_AM_B: return n / 8;
    case OP_BASE_CDFT2: return 4;
    case OP_BASE_PAIR2: return 2;
    case OP_BASE_OO8: return 1;
    case OP_CHAIN_F: case OP_CHAIN_B: return 1;
  }
  return 0;
}

OpCount ei_ops(const EI& e) {
  OpCount c;
  const uint64_t n = e.n;
  switch (e.op) {
    case OP_SC_B: c.adds = 2 * n - 4; break;
    case OP_SR_F: c.adds = n - 2; break;
    case OP_SH_F_DCT: case OP_ST_B_DCT: c.adds = n / 2; break;
    case OP_SH_F_DST: case OP_ST_B_DST: c.adds = n / 2 - 2; break;
    case OP_SH_F_ODD: case OP_ST_B_ODD: c.adds = n / 4; break;
    case OP_AM_F:
      if (e.am == 2 || e.am == 6) c.adds = n / 8 - 1; else c.muls = n / 8;
      break;
    case OP_AM_B:
      if (e.am == 4 || e.am == 8) c.adds = n / 8 - 1; else c.muls = n / 8;
      break;
    case OP_CHAIN_F: case OP_CHAIN_B: c.adds = e.aux - 1; c.bt = 1; break;
    case OP_BASE_CDFT2: c.adds = 4; break;
    case OP_BASE_PAIR2: c.adds = 2; break;
    case OP_BASE_OO8: c.muls = 1; break;
    default: break;
  }
  return c;
}

namespace {

EI mk(uint8_t op, uint8_t lens, uint32_t n, uint32_t off, uint32_t aux = 0,
      uint8_t am = 0, uint8_t flags = 0) {
  EI e;
  e.op = op;
  e.lens = lens;
  e.flags = flags;
  e.am = am;
  e.n = n;
  e.off = off;
  e.aux = aux;
  return e;
}

// The forward and backward EIs of one non-base node, and its children.
struct NodeSteps {
  EI fwd, bwd;
  int nchild = 0;
  int cf[2];
  size_t cn[2];
  uint32_t coff[2];
};

class Wiring {
 public:
  explicit Wiring(int v) : v_(v), tm_(time_major(v)), sine_(v >= 5) {}

  int dct_odd() const { return tm_ ? kDctOddTime : kDctOddHarm; }
  int dst_odd() const { return tm_ ? kDstOddTime : kDstOddHarm; }

  // Base-case EI of function f at its base size; false for pure copies.
  bool base(int f, uint32_t off, EI* out) const {
    switch (f) {
      case kCdft: *out = mk(OP_BASE_CDFT2, 0, 2, off); return true;
      case kRdft: case kDct: *out = mk(OP_BASE_PAIR2, 0, 2, off); return true;
      case kDctOddOdd: case kDstOddOdd: *out = mk(OP_BASE_OO8, 0, 8, off); return true;
      default: return false;  // Dst(4), odd(4): S = s (variants.cpp:373-387)
    }
  }

  NodeSteps steps(int f, size_t n, uint32_t off) const {
    NodeSteps s;
    const uint32_t N = static_cast<uint32_t>(n);
    switch (f) {
      case kCdft:
        s.fwd = mk(OP_SC_F, 0, N, off);
        s.bwd = mk(OP_SC_B, 0, N, off);
        s.nchild = 2;
        s.cf[0] = s.cf[1] = kRdft;
        s.cn[0] = s.cn[1] = n;
        s.coff[0] = off;
        s.coff[1] = off + N;
        return s;
      case kRdft:
        s.fwd = mk(OP_SR_F, 0, N, off);
        s.bwd = mk(OP_SR_B, 0, N, off);
        s.nchild = 2;
        s.cf[0] = kDct; s.cn[0] = n; s.coff[0] = off;
        s.cf[1] = kDst; s.cn[1] = n; s.coff[1] = off + N / 2 + 1;
        return s;
      case kDct: {
        const uint32_t ce = N / 4 + 1;
        if (tm_) {  // SplitTimeParity + HalveEvenTime
          s.fwd = mk(OP_GATHER, 0, N / 2 + 1, off, ce);
          s.bwd = mk(OP_ST_B_DCT, 0, N, off);
        } else {    // SplitHarmonicParity + HalveEvenHarmonics
          s.fwd = mk(OP_SH_F_DCT, 0, N, off);
          s.bwd = mk(OP_SCATTER, 0, N / 2 + 1, off, ce);
        }
        s.nchild = 2;
        s.cf[0] = kDct; s.cn[0] = n / 2; s.coff[0] = off;
        s.cf[1] = dct_odd(); s.cn[1] = n; s.coff[1] = off + ce;
        return s;
      }
      case kDst: {
        const uint32_t ce = N / 4 - 1;
        if (tm_) {
          s.fwd = mk(OP_GATHER, 1, N / 2 - 1, off, ce);
          s.bwd = mk(OP_ST_B_DST, 1, N, off);
        } else {
          s.fwd = mk(OP_SH_F_DST, 1, N, off);
          s.bwd = mk(OP_SCATTER, 1, N / 2 - 1, off, ce);
        }
        s.nchild = 2;
        s.cf[0] = kDst; s.cn[0] = n / 2; s.coff[0] = off;
        s.cf[1] = dst_odd(); s.cn[1] = n; s.coff[1] = off + ce;
        return s;
      }
      case kDctOddTime: case kDstOddTime: case kDctOddHarm: case kDstOddHarm: {
        const uint8_t lens = (f == kDstOddTime || f == kDstOddHarm) ? 1 : 0;
        const uint32_t mc = N / 4, ce = N / 8;
        if (tm_) {  // odd-time mother: SplitHarmonicParity + HalveEvenHarmonics
          s.fwd = mk(OP_SH_F_ODD, lens, N, off);
          s.bwd = mk(OP_SCATTER, lens, mc, off, ce);
        } else {    // odd-harmonic mother: SplitTimeParity + HalveEvenTime
          s.fwd = mk(OP_GATHER, lens, mc, off, ce);
          s.bwd = mk(OP_ST_B_ODD, lens, N, off);
        }
        s.nchild = 2;
        s.cf[0] = f; s.cn[0] = n / 2; s.coff[0] = off;
        s.cf[1] = lens ? kDstOddOdd : kDctOddOdd; s.cn[1] = n; s.coff[1] = off + ce;
        return s;
      }
      default: {  // odd-odd: AM conversion; child = odd function at n/2
        const uint8_t lens = f == kDstOddOdd ? 1 : 0;
        const uint8_t child_lens = sine_ ? static_cast<uint8_t>(1 - lens) : lens;
        const uint32_t q = N / 8;
        const int m = v_;
        if (m == 3 || m == 7) {
          // M3 dct: desc/sub, dst: asc/sub; M7 dct: asc/add, dst: desc/add
          uint8_t fl = 0;
          if ((m == 3 && lens == 0) || (m == 7 && lens == 1)) fl |= FL_DESC;
          if (m == 7) fl |= FL_ADD;
          s.fwd = mk(OP_CHAIN_F, lens, N, off, q, static_cast<uint8_t>(m), fl);
        } else {
          s.fwd = mk(OP_AM_F, lens, N, off, q, static_cast<uint8_t>(m));
        }
        if (m == 1 || m == 5) {
          // M1 dct: asc/sub, dst: desc/sub; M5 dct: desc/add, dst: asc/add
          uint8_t fl = 0;
          if ((m == 1 && lens == 1) || (m == 5 && lens == 0)) fl |= FL_DESC;
          if (m == 5) fl |= FL_ADD;
          s.bwd = mk(OP_CHAIN_B, lens, N, off, q, static_cast<uint8_t>(m), fl);
        } else {
          s.bwd = mk(OP_AM_B, lens, N, off, q, static_cast<uint8_t>(m));
        }
        s.nchild = 1;
        s.cf[0] = child_lens ? dst_odd() : dct_odd();
        s.cn[0] = n / 2;
        s.coff[0] = off;
        return s;
      }
    }
  }

 private:
  int v_;
  bool tm_, sine_;
};

// Single-CTA stage program of the subtree rooted at (f, n).
struct ProgBuilder {
  const Wiring& w;
  std::vector<std::pair<int, EI>> timed;

  // Returns the first free time slot after the node's last EI.
  int node(int f, size_t n, uint32_t off, int t) {
    if (n == fn_base(f)) {
      EI e;
      if (w.base(f, off, &e)) {
        timed.emplace_back(t, e);
        return t + 1;
      }
      return t;
    }
    const NodeSteps s = w.steps(f, n, off);
    timed.emplace_back(t, s.fwd);
    int end = t + 1;
    for (int c = 0; c < s.nchild; ++c)
      end = std::max(end, node(s.cf[c], s.cn[c], s.coff[c], t + 1));
    timed.emplace_back(end, s.bwd);
    return end + 1;
  }

  SubProgram build(int f, size_t n) {
    timed.clear();
    const int T = node(f, n, 0, 0);
    SubProgram p;
    p.fn = f;
    p.n = n;
    p.cells = fn_cells(f, n);
    std::stable_sort(timed.begin(), timed.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    size_t i = 0;
    for (int t = 0; t < T; ++t) {
      Stage st{static_cast<uint32_t>(p.eis.size()), 0, 0};
      uint32_t items = 0;
      for (; i < timed.size() && timed[i].first == t; ++i) {
        p.eis.push_back(timed[i].second);
        p.prefix.push_back(items);
        items += ei_items(timed[i].second);
        if (timed[i].second.op == OP_CHAIN_F || timed[i].second.op == OP_CHAIN_B)
          p.has_chain = 1;
      }
      st.ei_end = static_cast<uint32_t>(p.eis.size());
      st.items = items;
      if (st.ei_end > st.ei_begin) {
        p.stages.push_back(st);
        p.max_items = std::max(p.max_items, items);
      }
    }
    return p;
  }
};

// Multi-pass builder: nodes above the capacity become global EIs with
// explicit A/B buffer routing; subtrees within it become CTA jobs.
struct GlobalBuilder {
  const Wiring& w;
  size_t capacity;
  Compiled& out;
  std::map<std::pair<int, size_t>, uint32_t> prog_ids;
  std::vector<std::pair<int, EI>> fwd, bwd;

  uint32_t prog_for(int f, size_t n) {
    const auto key = std::make_pair(f, n);
    auto it = prog_ids.find(key);
    if (it != prog_ids.end()) return it->second;
    ProgBuilder pb{w, {}};
    out.progs.push_back(pb.build(f, n));
    const uint32_t id = static_cast<uint32_t>(out.progs.size() - 1);
    prog_ids[key] = id;
    return id;
  }

  // s: buffer holding the node's temporal cells; e: buffer that must hold
  // its spectrum.  Returns the backward height (0 for jobs).
  int node(int f, size_t n, uint32_t off, int t, uint8_t s, uint8_t e) {
    if (fn_cells(f, n) <= capacity || n == fn_base(f)) {
      out.jobs.push_back(Job{prog_for(f, n), off, s, e});
      return 0;
    }
    const NodeSteps st = w.steps(f, n, off);
    EI fe = st.fwd;
    fe.flags |= (s ? FL_SRC_B : 0) | (s ? 0 : FL_DST_B);
    fwd.emplace_back(t, fe);
    int h = 0;
    for (int c = 0; c < st.nchild; ++c)
      h = std::max(h, node(st.cf[c], st.cn[c], st.coff[c], t + 1,
                           static_cast<uint8_t>(1 - s), static_cast<uint8_t>(1 - e)));
    EI be = st.bwd;
    be.flags |= (e ? 0 : FL_SRC_B) | (e ? FL_DST_B : 0);
    bwd.emplace_back(h, be);
    return h + 1;
  }
};

void to_stages(std::vector<std::pair<int, EI>>& timed, std::vector<EI>& eis,
               std::vector<Stage>& stages) {
  std::stable_sort(timed.begin(), timed.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  size_t i = 0;
  while (i < timed.size()) {
    const int t = timed[i].first;
    Stage st{static_cast<uint32_t>(eis.size()), 0, 0};
    for (; i < timed.size() && timed[i].first == t; ++i) {
      eis.push_back(timed[i].second);
      st.items += ei_items(timed[i].second);
    }
    st.ei_end = static_cast<uint32_t>(eis.size());
    stages.push_back(st);
  }
}

void accumulate(OpCount& acc, const OpCount& c, uint64_t times = 1) {
  acc.adds += c.adds * times;
  acc.muls += c.muls * times;
  acc.bt += c.bt * times;
}

}  // namespace

Compiled compile(int variant, int fn, size_t n, size_t capacity_cells) {
  if (variant < 1 || variant > 8) fail("variant number must be in 1..8");
  if (fn < 0 || fn >= kNumFn) fail("unknown function");
  if (!fn_wired(variant, fn)) fail("variant does not wire this function");
  if (!is_pow2(n) || n < fn_base(fn))
    fail("periodization must be a power of two >= the function's base size");
  if (n > (size_t(1) << 31)) fail("periodization too large");
  const Wiring w(variant);
  Compiled c;
  c.variant = variant;
  c.fn = fn;
  c.n = n;
  c.cells = fn_cells(fn, n);
  if (c.cells <= capacity_cells) {
    ProgBuilder pb{w, {}};
    c.progs.push_back(pb.build(fn, n));
    c.single = true;
    for (const EI& e : c.progs[0].eis) accumulate(c.ops, ei_ops(e));
    return c;
  }
  c.single = false;
  c.root_src = 0;
  c.root_dst = 0;
  GlobalBuilder gb{w, capacity_cells, c, {}, {}, {}};
  gb.node(fn, n, 0, 0, c.root_src, c.root_dst);
  to_stages(gb.fwd, c.global_eis, c.fwd_stages);
  to_stages(gb.bwd, c.global_eis, c.bwd_stages);
  for (const EI& e : c.global_eis) accumulate(c.ops, ei_ops(e));
  for (const Job& j : c.jobs)
    for (const EI& e : c.progs[j.prog].eis) accumulate(c.ops, ei_ops(e));
  return c;
}

}  // namespace amqft_b200

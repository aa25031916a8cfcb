// bank_model.cpp -- DIAGNOSTIC: shared-memory bank model of the fast
// kernel's generated phases.  Compiles gen/fast_gen.cuh (build-time generated) as host C++ with a
// tracking value type: every read/write of a shared-buffer cell is logged
// per thread; threads are grouped into warps exactly as k_fast maps them,
// and each memory instruction (k-th access of the straight-line code) is
// scored in wavefronts = max over banks of distinct words.
//
//   g++ -O1 -std=c++17 -o /tmp/bank_model tools/bank_model.cpp && /tmp/bank_model 4 12
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <vector>
#define __device__
#define __forceinline__ inline
#define __ldg(p) (*(p))
#ifndef AMQFT_CHAIN_SHIFT
#define AMQFT_CHAIN_SHIFT 1
#endif

struct Acc { long addr; bool wr; };
static std::vector<Acc>* g_tr = nullptr;
static const void* g_lo = nullptr;
static const void* g_hi = nullptr;

struct TR {
  double v = 0;
  TR() = default;
  TR(double x) : v(x) {}
  TR(const TR& o) : v(o.v) { rec(&o, false); }
  TR& operator=(const TR& o) { rec(this, true); v = o.v; return *this; }
  static void rec(const TR* p, bool wr) {
    if (g_tr && (const void*)p >= g_lo && (const void*)p < g_hi)
      g_tr->push_back({(long)(p - (const TR*)g_lo), wr});
  }
};
struct TA {
  static TR add(TR a, TR b) { return TR(a.v + b.v); }
  static TR sub(TR a, TR b) { return TR(a.v - b.v); }
  static TR mul(TR a, TR b) { return TR(a.v * b.v); }
};

#include "../paper_1404_1810_b200/csrc/gen/fast_gen.cuh"
using namespace amqft_b200;

static int V_, LOGN, N, H, LB = 64, LOGLB = 6, LT, HP, NSEG, CS, SINE;
static bool TM;
#ifndef AMQFT_CHAIN_SHIFT_F
#define AMQFT_CHAIN_SHIFT_F AMQFT_CHAIN_SHIFT
#endif
// kernel scheme (Cfg::coT / coF): skewed buffer shift 1, padded buffer 16;
// -DAMQFT_CHAIN_SHIFT / _F override both
static int co(int c) {
#ifdef AMQFT_CHAIN_SHIFT_OVERRIDE
  return c * CS + (c >> 1) * AMQFT_CHAIN_SHIFT;
#else
  return c * CS + (c >> 1) * (TM ? 1 : 16);
#endif
}
static int cf(int c) {
#ifdef AMQFT_CHAIN_SHIFT_OVERRIDE
  return c * CS + (c >> 1) * AMQFT_CHAIN_SHIFT_F;
#else
  return c * CS + (c >> 1) * (TM ? 16 : 1);
#endif
}
static int skew(int i) { return i + (i >> LOGLB); }
static int swz(int i, int lam) { return i + ((i + (lam ? 0 : 31)) >> 5); }
static int parity(unsigned x) { return __builtin_popcount(x) & 1; }

static void seg_params(int lam_c, int s, int d, int* rho, int* lens, int* r) {
  *rho = d == 0 ? 0 : (s & 1);
  *lens = lam_c ^ (SINE & parity(static_cast<unsigned>(s ^ (s >> 1))));
  int res = 0, ln = lam_c, prev = 0;
  for (int i = 1; i <= d; ++i) {
    const int b = (s >> (d - i)) & 1;
    const int is_o = b != prev;
    res |= (is_o ^ ln) << (i - 1);
    ln ^= SINE & is_o;
    prev = b;
  }
  *r = res;
}

// Score: traces[tid] for NT threads; warp w = tids 32w..32w+31.
static void score(const char* name, std::vector<std::vector<Acc>>& tr, int nt) {
  long wf = 0, ideal = 0, insts = 0, mism = 0, exw = 0;
  for (int w = 0; w < nt / 32; ++w) {
    size_t len = 0;
    for (int l = 0; l < 32; ++l) len = std::max(len, tr[w * 32 + l].size());
    for (size_t k = 0; k < len; ++k) {
      std::map<int, std::set<long>> banks;
      int active = 0;
      for (int l = 0; l < 32; ++l) {
        auto& t = tr[w * 32 + l];
        if (k < t.size()) { banks[t[k].addr & 31].insert(t[k].addr); ++active; }
      }
      if (active != 32 && active != 0) ++mism;
      size_t m = 0;
      for (auto& b : banks) m = std::max(m, b.second.size());
      wf += m;
      if (tr[w * 32].size() > k && tr[w * 32][k].wr) exw += m - 1;
      ideal += 1;
      ++insts;
    }
  }
  printf("%-10s warp-insts %6ld wavefronts %6ld (excess %5ld, writes %5ld) partial-warp insts %ld\n", name, insts,
         wf, wf - ideal, exw, mism);
}

template <int V, int LOGN_>
static void run_all() {
  constexpr int N_ = 1 << LOGN_, H_ = N_ / 2, LT_ = LOGN_ - 1 - 6, HP_ = H_ / 64;
  std::vector<TR> sm(16 * CS + 64), tab(N_ * 4, TR(0.5));
  TR* Tb = sm.data();
  TR* Fb = Tb + 4 * CS;
  g_lo = sm.data();
  g_hi = sm.data() + sm.size();
  const int NT = 256;
  std::vector<std::vector<Acc>> tr(NT);
  // ---- top (TM fwd) or fold (HM)
  for (auto& t : tr) t.clear();
  for (int tid = 0; tid < NT; ++tid) {
    g_tr = &tr[tid];
    if (TM) {
      const int c = tid >> 6, v = tid & 63;
      if (v > 0) Top<64, LT_, LOGN_, (V >= 5)>::template fwd<TR, TA>(c & 1, Tb + co(c), v, tab.data(), TR(0.5));
    } else if (tid < 128 && (tid & 31)) {
      Recomb<64, H_ / 64>::template fold<TR, TA>((tid >> 5) & 1, Tb + co(tid >> 5), tid & 31);
    }
  }
  score(TM ? "top" : "fold", tr, NT);
  // ---- bottom
  for (int part = 0; part < 2; ++part) {
    for (auto& t : tr) t.clear();
    for (int tid = 0; tid < NSEG; ++tid) {
      g_tr = &tr[tid];
      const int half = HP_ / 2, h = tid % half, rest = tid / half;
      const int p = rest & 1, rho_bit = (rest >> 1) & 1, lam_bit = (rest >> 2) & 1;
      const int c = p * 2 + lam_bit, s = 2 * h + rho_bit;
      int rho, lens, r;
      seg_params(lam_bit, s, LT_, &rho, &lens, &r);
      if (part == 0)
        Bottom<V, 64>::template run<TR, TA, 6, LT_, 0>(rho, lens, Tb + co(c), Fb + cf(c), s * 64, tab.data(), N_,
                                                       TR(0.5), N_, r, lam_bit);
      else
        Bottom<V, 64>::template run<TR, TA, 6, LT_, 1>(rho, lens, Tb + co(c), Fb + cf(c), s * 64, tab.data(), N_,
                                                       TR(0.5), N_, r, lam_bit);
    }
    score(part == 0 ? "bottom p0" : "bottom p1", tr, NSEG);
  }
  // ---- recomb (TM) or top bwd (HM)
  for (auto& t : tr) t.clear();
  for (int tid = 0; tid < NT; ++tid) {
    g_tr = &tr[tid];
    if (TM) {
      if (tid < 128 && (tid & 31))
        Recomb<64, H_ / 64>::template run<TR, TA>((tid >> 5) & 1, Fb + cf(tid >> 5), tid & 31);
    } else {
      const int c = tid >> 6, v = tid & 63;
      if (v > 0) Top<64, LT_, LOGN_, (V >= 5)>::template bwd<TR, TA>(c & 1, Fb + cf(c), v, tab.data(), TR(0.5));
    }
  }
  score(TM ? "recomb" : "top bwd", tr, NT);
  g_tr = nullptr;
}

int main(int argc, char** argv) {
  V_ = argc > 1 ? atoi(argv[1]) : 4;
  LOGN = argc > 2 ? atoi(argv[2]) : 12;
  N = 1 << LOGN; H = N / 2; LT = LOGN - 1 - LOGLB; HP = H / LB; NSEG = 4 * HP;
  CS = ((H + HP + 1 > H + H / 32 + 1 ? H + HP + 1 : H + H / 32 + 1) + 31) / 32 * 32 + 16;
  TM = V_ == 1 || V_ == 4 || V_ == 5 || V_ == 8;
  SINE = V_ >= 5;
  printf("v%d N=%d shift=%d\n", V_, N, AMQFT_CHAIN_SHIFT);
  if (LOGN != 12) { printf("only N=4096 wired\n"); return 1; }
  switch (V_) {
    case 1: run_all<1, 12>(); break;
    case 2: run_all<2, 12>(); break;
    case 3: run_all<3, 12>(); break;
    case 4: run_all<4, 12>(); break;
    case 5: run_all<5, 12>(); break;
    case 6: run_all<6, 12>(); break;
    case 7: run_all<7, 12>(); break;
    case 8: run_all<8, 12>(); break;
  }
  return 0;
}

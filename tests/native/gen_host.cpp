// gen_host.cpp -- TEST HARNESS: compiles the generated device code
// (paper_1404_1810_b200/csrc/gen/fast_gen.cuh, generated at build time) as host C++ so the CPU test
// suite can check every generated function against the fast-kernel model
// (tests/fast_model.py) without a GPU.  fp64, -ffp-contract=off.
#define __device__
#define __forceinline__ inline
#define __ldg(p) (*(p))
#include "../../paper_1404_1810_b200/csrc/gen/fast_gen.cuh"

namespace {
struct HA {
  static double add(double a, double b) { return a + b; }
  static double sub(double a, double b) { return a - b; }
  static double mul(double a, double b) { return a * b; }
};
using namespace amqft_b200;
}  // namespace

template <int V>
int bottom_v(int LB, int rho, int lens, const double* T, double* F, int a, const double* tab,
             int nmax, double base, int N, int D, int r, int dsto) {
  if (LB != 64) return -1;
  switch (D) {
    case 3:
      if (rho != 0) return -1;   // odd segments are stored reversed: orientation 0 only
      Bottom<V, 64>::template run<double, HA, 6, 3, 2>(rho, lens, T, F, a, tab, nmax, base, N, r, dsto);
      return 0;
    case 4:
      if (rho != 0) return -1;   // odd segments are stored reversed: orientation 0 only
      Bottom<V, 64>::template run<double, HA, 6, 4, 2>(rho, lens, T, F, a, tab, nmax, base, N, r, dsto);
      return 0;
    case 5:
      if (rho != 0) return -1;   // odd segments are stored reversed: orientation 0 only
      Bottom<V, 64>::template run<double, HA, 6, 5, 2>(rho, lens, T, F, a, tab, nmax, base, N, r, dsto);
      return 0;
    case 6:
      if (rho != 0) return -1;   // odd segments are stored reversed: orientation 0 only
      Bottom<V, 64>::template run<double, HA, 6, 6, 2>(rho, lens, T, F, a, tab, nmax, base, N, r, dsto);
      return 0;
  }
  return -1;
}

template <int V, int HP, int NL>
int small_vh(int LB, int lam, const double* T, double* F, const double* tab, double base) {
  if (LB == 64) { SmallFull<V, HP, NL>::template run<double, HA, 6, 64>(lam, T, F, tab, base); return 0; }
  return -1;
}

template <int V>
int small_v(int HP, int nlog, int LB, int lam, const double* T, double* F, const double* tab,
            double base) {
  if (HP == 8 && nlog == 10) return small_vh<V, 8, 10>(LB, lam, T, F, tab, base);
  if (HP == 16 && nlog == 11) return small_vh<V, 16, 11>(LB, lam, T, F, tab, base);
  if (HP == 32 && nlog == 12) return small_vh<V, 32, 12>(LB, lam, T, F, tab, base);
  if (HP == 64 && nlog == 13) return small_vh<V, 64, 13>(LB, lam, T, F, tab, base);
  return -1;
}


template <int V>
int smallpar_v(int HP, int nlog, int LB, int lam, int cls, const double* T, double* F,
               const double* tab, double base, int serial, double* B) {
  if (LB != 64) return -1;
#define SPCASE(hp, nl)                                                                      \
  if (HP == hp && nlog == nl) {                                                             \
    if (serial) SmallPar<V, hp, nl>::template serial<double, HA>(lam, B);                   \
    else SmallPar<V, hp, nl>::template cls<double, HA, 6, 64>(lam, cls, T, F, tab, base);   \
    return 0;                                                                               \
  }
  SPCASE(8, 10) SPCASE(16, 11) SPCASE(32, 12) SPCASE(64, 13)
#undef SPCASE
  return -1;
}


extern "C" {

int host_top(int LB, int LT, int nlog, int sine, int bwd, int lam, double* B, int v,
             const double* tab, double base) {
#define TOPCASE(lb, lt, nl)                                                        \
  if (LB == lb && LT == lt && nlog == nl) {                                         \
    if (sine) {                                                                     \
      if (bwd) Top<lb, lt, nl, 1>::bwd<double, HA>(lam, B, v, tab, base);           \
      else Top<lb, lt, nl, 1>::fwd<double, HA>(lam, B, v, tab, base);               \
    } else {                                                                        \
      if (bwd) Top<lb, lt, nl, 0>::bwd<double, HA>(lam, B, v, tab, base);           \
      else Top<lb, lt, nl, 0>::fwd<double, HA>(lam, B, v, tab, base);               \
    }                                                                               \
    return 0;                                                                       \
  }
  TOPCASE(64, 3, 10) TOPCASE(64, 4, 11) TOPCASE(64, 5, 12) TOPCASE(64, 6, 13)
#undef TOPCASE
  return -1;
}

int host_bottom(int V, int LB, int rho, int lens, const double* T, double* F, int a,
                const double* tab, int nmax, double base, int N, int D, int r, int dsto) {
  switch (V) {
    case 1: return bottom_v<1>(LB, rho, lens, T, F, a, tab, nmax, base, N, D, r, dsto);
    case 2: return bottom_v<2>(LB, rho, lens, T, F, a, tab, nmax, base, N, D, r, dsto);
    case 3: return bottom_v<3>(LB, rho, lens, T, F, a, tab, nmax, base, N, D, r, dsto);
    case 4: return bottom_v<4>(LB, rho, lens, T, F, a, tab, nmax, base, N, D, r, dsto);
    case 5: return bottom_v<5>(LB, rho, lens, T, F, a, tab, nmax, base, N, D, r, dsto);
    case 6: return bottom_v<6>(LB, rho, lens, T, F, a, tab, nmax, base, N, D, r, dsto);
    case 7: return bottom_v<7>(LB, rho, lens, T, F, a, tab, nmax, base, N, D, r, dsto);
    case 8: return bottom_v<8>(LB, rho, lens, T, F, a, tab, nmax, base, N, D, r, dsto);
  }
  return -1;
}

int host_small(int V, int HP, int nlog, int LB, int lam, const double* T, double* F,
               const double* tab, double base) {
  switch (V) {
    case 1: return small_v<1>(HP, nlog, LB, lam, T, F, tab, base);
    case 2: return small_v<2>(HP, nlog, LB, lam, T, F, tab, base);
    case 3: return small_v<3>(HP, nlog, LB, lam, T, F, tab, base);
    case 4: return small_v<4>(HP, nlog, LB, lam, T, F, tab, base);
    case 5: return small_v<5>(HP, nlog, LB, lam, T, F, tab, base);
    case 6: return small_v<6>(HP, nlog, LB, lam, T, F, tab, base);
    case 7: return small_v<7>(HP, nlog, LB, lam, T, F, tab, base);
    case 8: return small_v<8>(HP, nlog, LB, lam, T, F, tab, base);
  }
  return -1;
}

int host_smallpar(int V, int HP, int nlog, int LB, int lam, int cls, const double* T, double* F,
                  const double* tab, double base, int serial, double* B) {
  switch (V) {
    case 1: return smallpar_v<1>(HP, nlog, LB, lam, cls, T, F, tab, base, serial, B);
    case 2: return smallpar_v<2>(HP, nlog, LB, lam, cls, T, F, tab, base, serial, B);
    case 3: return smallpar_v<3>(HP, nlog, LB, lam, cls, T, F, tab, base, serial, B);
    case 4: return smallpar_v<4>(HP, nlog, LB, lam, cls, T, F, tab, base, serial, B);
    case 5: return smallpar_v<5>(HP, nlog, LB, lam, cls, T, F, tab, base, serial, B);
    case 6: return smallpar_v<6>(HP, nlog, LB, lam, cls, T, F, tab, base, serial, B);
    case 7: return smallpar_v<7>(HP, nlog, LB, lam, cls, T, F, tab, base, serial, B);
    case 8: return smallpar_v<8>(HP, nlog, LB, lam, cls, T, F, tab, base, serial, B);
  }
  return -1;
}

#define RECOMB_SIZES(X) X(64, 8) X(64, 16) X(64, 32) X(128, 32)
int host_recomb(int W, int HW, int lam, double* F, int k) {
#define X(w, hw) if (W == w && HW == hw) { Recomb<w, hw>::run<double, HA>(lam, F, k); return 0; }
  RECOMB_SIZES(X)
#undef X
  return -1;
}

int host_fold(int W, int HW, int lam, double* F, int k) {
#define X(w, hw) if (W == w && HW == hw) { Recomb<w, hw>::fold<double, HA>(lam, F, k); return 0; }
  RECOMB_SIZES(X)
#undef X
  return -1;
}

}  // extern "C"

// gll_host.cpp -- GLL nodes, weights and the Legendre analysis / synthesis matrices
// (DESIGN.md 3.1-3.2), built on the host in binary128 so that the single rounding
// to binary64 is correct (pinned against 40-digit decimal arithmetic by
// tests/golden/make_golden.py).  Nodes: +-1 and the roots of P'_N (N = lx-1) by
// Newton on x P_N - P_{N-1} = 0, mirrored exactly; weights 2/(N(N+1)P_N(x_i)^2);
// F[k][i] = w_i L_k(x_i)/sqrt(g_k), B[i][k] = L_k(x_i)/sqrt(g_k) with g_k = 2/(2k+1)
// (k < N) and g_N = 2/N (discrete GLL norm); parity (-1)^k enforced by mirroring.
#include <quadmath.h>

namespace isf {
namespace host {

typedef __float128 qreal;
constexpr int kMaxLxHost = 16;

static void legendre_q(int N, qreal x, qreal* P) {
  P[0] = 1;
  if (N >= 1) P[1] = x;
  for (int k = 2; k <= N; ++k) P[k] = ((qreal)(2 * k - 1) * x * P[k - 1] - (qreal)(k - 1) * P[k - 2]) / (qreal)k;
}

static void gll_nodes_q(int lx, qreal* x, qreal* w) {
  const int N = lx - 1;
  qreal P[kMaxLxHost + 1];
  for (int i = 0; i <= N; ++i) {
    const qreal pi = acosq((qreal)-1);
    qreal xi = -cosq(pi * (qreal)i / (qreal)N);
    for (int it = 0; it < 100; ++it) {
      legendre_q(N, xi, P);
      const qreal dx = (xi * P[N] - P[N - 1]) / ((qreal)(N + 1) * P[N]);
      xi -= dx;
      if (fabsq(dx) < (qreal)1e-33) break;
    }
    x[i] = xi;
  }
  x[0] = -1;
  x[N] = 1;
  for (int i = 0; i < lx / 2; ++i) x[N - i] = -x[i];
  if (lx % 2) x[lx / 2] = 0;
  for (int i = 0; i <= N; ++i) {
    legendre_q(N, x[i], P);
    w[i] = (qreal)2 / ((qreal)N * (qreal)(N + 1) * P[N] * P[N]);
  }
  for (int i = 0; i < lx / 2; ++i) w[N - i] = w[i];
}

void build_operators(int lx, double* F, double* B, double* xd, double* wd) {
  const int N = lx - 1;
  qreal x[kMaxLxHost], w[kMaxLxHost], P[kMaxLxHost + 1];
  gll_nodes_q(lx, x, w);
  for (int i = 0; i < lx; ++i) {
    if (xd) xd[i] = (double)x[i];
    if (wd) wd[i] = (double)w[i];
  }
  for (int i = 0; i < (lx + 1) / 2; ++i) {
    legendre_q(N, x[i], P);
    for (int k = 0; k < lx; ++k) {
      const qreal g = (k < N) ? (qreal)2 / (qreal)(2 * k + 1) : (qreal)2 / (qreal)N;
      const qreal rs = 1 / sqrtq(g);
      double f = (double)(w[i] * P[k] * rs);
      double b = (double)(P[k] * rs);
      if ((lx % 2) && i == lx / 2 && (k % 2)) { f = 0.0; b = 0.0; }
      F[k * lx + i] = f;
      B[i * lx + k] = b;
      if (i != N - i) {
        F[k * lx + (N - i)] = (k % 2) ? -f : f;
        B[(N - i) * lx + k] = (k % 2) ? -b : b;
      }
    }
  }
}

}  // namespace host
}  // namespace isf

// oracle.cpp — plain, slow, serial CPU oracle for the sunbw hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
// The product (paper_2011_12984_b200/) never links, imports or calls it, and
// it shares no header, kernel, helper, table or constant with the CUDA path.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -fPIC -shared
// (x86-64 SSE2 double arithmetic: every + - * / sqrt is one IEEE RN-even
// rounding; -ffp-contract=off forbids FMA contraction; denormals are on).
//
// Citation key: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
// "DESIGN Rk" = reading k listed in DESIGN.md §3 (taken from SURVEY §8(c)).
//
// Every function states the passage it follows.  Where the paper defines an
// operation only by name (the N_Vector roster), the oracle is
// the plain mathematical definition written out in index order.
//
// Parity status: every function here is pinned by tests/test_oracle_*.py
// (closed forms, brute force, exact rational arithmetic, textbook reductions).
// The paper prints no solution values for the nonlinear Brusselator (P:425-486
// are figure placeholders); its SBDF trajectory is pinned to an independent
// integrator instead (scipy Radau IIA on the semi-discrete system written out
// from P:369-371: second-order convergence to it, error < 1e-5 at h = 1e-3).

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

extern "C" {

// ---------------------------------------------------------------------------
// O1 streaming operations ("streaming operations like adding two vectors
// or scaling a vector"; roster S:129-141).  One IEEE rounding per operation,
// no contraction, no special-casing of coefficients (DESIGN R3).
// ---------------------------------------------------------------------------

void oracle_linear_sum(int64_t n, double a, const double* x, double b,
                       const double* y, double* z) {
  for (int64_t i = 0; i < n; ++i) {
    double ax = a * x[i];
    double by = b * y[i];
    z[i] = ax + by;
  }
}

void oracle_scale(int64_t n, double c, const double* x, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = c * x[i];
}

void oracle_prod(int64_t n, const double* x, const double* y, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = x[i] * y[i];
}

void oracle_div(int64_t n, const double* x, const double* y, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = x[i] / y[i];
}

void oracle_const(int64_t n, double c, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = c;
}

void oracle_abs(int64_t n, const double* x, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = std::fabs(x[i]);
}

void oracle_inv(int64_t n, const double* x, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = 1.0 / x[i];
}

void oracle_add_const(int64_t n, const double* x, double b, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = x[i] + b;
}

// ---------------------------------------------------------------------------
// O2 reductions ("reduction operations, like norms or dot products";
// P:180-182 scalar result returned to the host).
// The sum is a Neumaier-compensated left fold (DESIGN R6): a plain left fold
// has relative error ~1e-12 at n=1e9, above the parity bar.
// ---------------------------------------------------------------------------

struct Neumaier {
  double s = 0.0, c = 0.0;
  void add(double t) {
    double tt = s + t;
    if (std::fabs(s) >= std::fabs(t))
      c += (s - tt) + t;
    else
      c += (t - tt) + s;
    s = tt;
  }
  double value() const { return s + c; }
};

// Σ x_i y_i  (N_VDotProd; global = this over the concatenation)
double oracle_dot(int64_t n, const double* x, const double* y) {
  Neumaier acc;
  for (int64_t i = 0; i < n; ++i) acc.add(x[i] * y[i]);
  return acc.value();
}

// Σ (x_i w_i)^2 — the local partial of the WRMS norm (N_VWSqrSumLocal)
double oracle_wsqrsum(int64_t n, const double* x, const double* w) {
  Neumaier acc;
  for (int64_t i = 0; i < n; ++i) {
    double p = x[i] * w[i];
    acc.add(p * p);
  }
  return acc.value();
}

// Σ_{id_i>0} (x_i w_i)^2
double oracle_wsqrsum_mask(int64_t n, const double* x, const double* w,
                           const double* id) {
  Neumaier acc;
  for (int64_t i = 0; i < n; ++i) {
    if (id[i] > 0.0) {
      double p = x[i] * w[i];
      acc.add(p * p);
    }
  }
  return acc.value();
}

// sqrt(Σ (x_i w_i)^2 / N), N = n (DESIGN R5: global length, also under mask)
double oracle_wrms(int64_t n, const double* x, const double* w) {
  if (n <= 0) return std::nan("");
  double s = oracle_wsqrsum(n, x, w);
  return std::sqrt(s / (double)n);
}

double oracle_wrms_mask(int64_t n, const double* x, const double* w,
                        const double* id) {
  if (n <= 0) return std::nan("");
  double s = oracle_wsqrsum_mask(n, x, w, id);
  return std::sqrt(s / (double)n);
}

// max |x_i|; NaN never selected (predicate |x|>max, DESIGN R9); n=0 → NaN
double oracle_max_norm(int64_t n, const double* x) {
  if (n <= 0) return std::nan("");
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double a = std::fabs(x[i]);
    if (a > m) m = a;
  }
  return m;
}

// min x_i; n=0 → +inf (identity of min; the global op errors on N=0)
double oracle_min(int64_t n, const double* x) {
  double m = INFINITY;
  for (int64_t i = 0; i < n; ++i)
    if (x[i] < m) m = x[i];
  return m;
}

// ---------------------------------------------------------------------------
// O3 fused operations (not in the paper; SUNDIALS definitions, DESIGN R1/R4).
// ---------------------------------------------------------------------------

// z = Σ_j c_j X_j, summed left to right in j: z = c0 X0; z = z + c_j X_j.
void oracle_linear_combination(int nv, const double* c, const double* const* X,
                               int64_t n, double* z) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = c[0] * X[0][i];
    for (int j = 1; j < nv; ++j) {
      double t = c[j] * X[j][i];
      acc = acc + t;
    }
    z[i] = acc;
  }
}

// Z_j = a_j x + Y_j
void oracle_scale_add_multi(int nv, const double* a, const double* x,
                            const double* const* Y, double* const* Z,
                            int64_t n) {
  for (int j = 0; j < nv; ++j)
    for (int64_t i = 0; i < n; ++i) {
      double t = a[j] * x[i];
      Z[j][i] = t + Y[j][i];
    }
}

// d_j = x · Y_j
void oracle_dot_prod_multi(int nv, const double* x, const double* const* Y,
                           int64_t n, double* dots) {
  for (int j = 0; j < nv; ++j) dots[j] = oracle_dot(n, x, Y[j]);
}

// ---------------------------------------------------------------------------
// Block-diagonal matrix (square blocks A_j sharing one pattern).
// Storage: G blocks of m×m, row-major within a block, blocks contiguous.
// ---------------------------------------------------------------------------

// A <- c A + I  (SUNMatScaleAddI): a_ij = RN(c a_ij), then a_ii += 1.
void oracle_scale_add_identity(int64_t G, int m, double c, double* A) {
  for (int64_t g = 0; g < G; ++g) {
    double* a = A + g * m * m;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        double v = c * a[i * m + j];
        if (i == j) v = v + 1.0;
        a[i * m + j] = v;
      }
  }
}

// O6: LU with partial pivoting per block, in place (Doolittle, unit L below
// the diagonal, U on and above).  Column k: pivot = first row of max |a_ik|,
// i >= k (LAPACK idamax rule, DESIGN R11); swap whole rows; l_ik = a_ik/a_kk;
// a_ij -= l_ik a_kj for j > k.  piv[g*m + k] = chosen row at step k (0-based).
// A zero pivot marks the block singular: elimination of that column is
// skipped and the block is finished.  Returns 1 + first singular block, or 0.
// (Role of cuSolverSp batch-QR; per-cell dense solve per P:389-390.)
int64_t oracle_lu_factor(int64_t G, int m, double* A, int32_t* piv) {
  int64_t first_singular = 0;
  for (int64_t g = 0; g < G; ++g) {
    double* a = A + g * m * m;
    int32_t* p = piv + g * m;
    bool singular = false;
    for (int k = 0; k < m; ++k) {
      int r = k;
      double best = std::fabs(a[k * m + k]);
      for (int i = k + 1; i < m; ++i) {
        double v = std::fabs(a[i * m + k]);
        if (v > best) { best = v; r = i; }
      }
      p[k] = r;
      if (r != k)
        for (int j = 0; j < m; ++j) {
          double t = a[k * m + j];
          a[k * m + j] = a[r * m + j];
          a[r * m + j] = t;
        }
      double akk = a[k * m + k];
      if (akk == 0.0) { singular = true; continue; }
      for (int i = k + 1; i < m; ++i) {
        double l = a[i * m + k] / akk;
        a[i * m + k] = l;
        for (int j = k + 1; j < m; ++j) {
          double t = l * a[k * m + j];
          a[i * m + j] = a[i * m + j] - t;
        }
      }
    }
    if (singular && first_singular == 0) first_singular = g + 1;
  }
  return first_singular;
}

// Block inverse by symbolic Gauss-Jordan (the paper's task-local solver,
// "applying the inverse of each 3x3 block matrix ... generated
// offline with a symbolic Gauss-Jordan method").  Gauss-Jordan on [A | I]
// WITHOUT pivoting (a symbolic elimination fixes the operation sequence),
// k = 0..m-1 in order:
//   p = RN(1/A_kk)                                 (pivot reciprocal)
//   A_kj = RN(A_kj p), j > k;  B_kj = RN(B_kj p)   (normalise the pivot row)
//   for i != k, f = A_ik:  A_ij = RN(A_ij - RN(f A_kj)), j > k
//                          B_ij = RN(B_ij - RN(f B_kj))
// "Symbolic": the right-hand block starts as the identity and the generator
// emits no operation on its structural zeros and ones — B_kj = 0 is not
// scaled or subtracted, a structural 1 times p is p, and 0 - RN(f B_kj) is
// -RN(f B_kj).  The left block is treated as dense.  B ends as A^{-1}.
// A zero pivot marks the block singular (first one returned, 1-based) and
// the sequence continues with IEEE arithmetic (1/0 = inf).
int64_t oracle_gj_inverse(int64_t G, int m, const double* Ain, double* Binv) {
  int64_t first_singular = 0;
  std::vector<double> A(m * m), B(m * m);
  std::vector<int> kind(m * m);   // B structure: 0 structural zero, 1 structural one, 2 value
  for (int64_t g = 0; g < G; ++g) {
    for (int e = 0; e < m * m; ++e) {
      A[e] = Ain[g * m * m + e];
      B[e] = (e % (m + 1) == 0) ? 1.0 : 0.0;
      kind[e] = (e % (m + 1) == 0) ? 1 : 0;
    }
    for (int k = 0; k < m; ++k) {
      if (A[k * m + k] == 0.0 && first_singular == 0) first_singular = g + 1;
      const double p = 1.0 / A[k * m + k];
      for (int j = k + 1; j < m; ++j) A[k * m + j] = A[k * m + j] * p;
      for (int j = 0; j < m; ++j) {
        if (kind[k * m + j] == 0) continue;
        B[k * m + j] = kind[k * m + j] == 1 ? p : B[k * m + j] * p;
        kind[k * m + j] = 2;
      }
      for (int i = 0; i < m; ++i) {
        if (i == k) continue;
        const double f = A[i * m + k];
        for (int j = k + 1; j < m; ++j) {
          double t = f * A[k * m + j];
          A[i * m + j] = A[i * m + j] - t;
        }
        for (int j = 0; j < m; ++j) {
          if (kind[k * m + j] == 0) continue;
          double t = f * B[k * m + j];
          if (kind[i * m + j] == 0) {
            B[i * m + j] = -t;
          } else {
            double bij = kind[i * m + j] == 1 ? 1.0 : B[i * m + j];
            B[i * m + j] = bij - t;
          }
          kind[i * m + j] = 2;
        }
      }
    }
    for (int e = 0; e < m * m; ++e) Binv[g * m * m + e] = B[e];
  }
  return first_singular;
}

// x = A^{-1} b per block with the inverse from oracle_gj_inverse: each row a
// left-to-right sum, x_i = RN(...RN(RN(B_i0 b_0) + RN(B_i1 b_1))... + RN(B_i,m-1 b_m-1)).
// x may alias b.
void oracle_gj_apply(int64_t G, int m, const double* Binv, const double* b, double* x) {
  std::vector<double> y(m);
  for (int64_t g = 0; g < G; ++g) {
    const double* B = Binv + g * m * m;
    for (int i = 0; i < m; ++i) {
      double s = B[i * m] * b[g * m];
      for (int j = 1; j < m; ++j) {
        double t = B[i * m + j] * b[g * m + j];
        s = s + t;
      }
      y[i] = s;
    }
    for (int i = 0; i < m; ++i) x[g * m + i] = y[i];
  }
}

// O7: x = U^{-1} L^{-1} P b per block; x may alias b.  Forward then back
// substitution in index order, each Σ as sequential RN subtractions.
void oracle_lu_solve(int64_t G, int m, const double* LU, const int32_t* piv,
                     const double* b, double* x) {
  std::vector<double> y(m);
  for (int64_t g = 0; g < G; ++g) {
    const double* a = LU + g * m * m;
    const int32_t* p = piv + g * m;
    for (int i = 0; i < m; ++i) y[i] = b[g * m + i];
    for (int k = 0; k < m; ++k) {
      int r = p[k];
      if (r != k) { double t = y[k]; y[k] = y[r]; y[r] = t; }
    }
    for (int i = 0; i < m; ++i) {
      double s = y[i];
      for (int j = 0; j < i; ++j) {
        double t = a[i * m + j] * y[j];
        s = s - t;
      }
      y[i] = s;
    }
    for (int i = m - 1; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < m; ++j) {
        double t = a[i * m + j] * y[j];
        s = s - t;
      }
      y[i] = s / a[i * m + i];
    }
    for (int i = 0; i < m; ++i) x[g * m + i] = y[i];
  }
}

// y = A x per block (the low-storage block SpMV role)
void oracle_block_matvec(int64_t G, int m, const double* A, const double* x,
                         double* y) {
  for (int64_t g = 0; g < G; ++g)
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int j = 0; j < m; ++j) {
        double t = A[g * m * m + i * m + j] * x[g * m + j];
        s = s + t;
      }
      y[g * m + i] = s;
    }
}

// ---------------------------------------------------------------------------
// Brusselator advection–reaction.  State interleaved per cell
// (u,v,w) (DESIGN R12).  Parameters: c, A, B, eps.
// ---------------------------------------------------------------------------

// O8 reaction f_I (reaction terms):
//   f_u = A - (w+1) u + v u^2 ;  f_v = w u - v u^2 ;  f_w = (B - w)/eps - w u
void oracle_bruss_reaction(int64_t G, const double* y, double A, double B,
                           double eps, double* f) {
  for (int64_t g = 0; g < G; ++g) {
    double u = y[3 * g], v = y[3 * g + 1], w = y[3 * g + 2];
    double uu = u * u;
    double vuu = v * uu;
    double w1 = w + 1.0;
    double w1u = w1 * u;
    double fu = A - w1u;
    fu = fu + vuu;
    double wu = w * u;
    double fv = wu - vuu;
    double bw = B - w;
    double bwe = bw / eps;
    double fw = bwe - wu;
    f[3 * g] = fu;
    f[3 * g + 1] = fv;
    f[3 * g + 2] = fw;
  }
}

// O5 reaction Jacobian J = ∂f_I/∂(u,v,w) (P:369-371 differentiated; P:389
// block structure), stored as G row-major 3×3 blocks.  inv_eps = RN(1/eps).
void oracle_bruss_jacobian(int64_t G, const double* y, double eps, double* J) {
  double inv_eps = 1.0 / eps;
  for (int64_t g = 0; g < G; ++g) {
    double u = y[3 * g], v = y[3 * g + 1], w = y[3 * g + 2];
    double uu = u * u;
    double u2 = 2.0 * u;
    double uv2 = u2 * v;
    double* a = J + 9 * g;
    double w1 = w + 1.0;
    a[0] = uv2 - w1;          // ∂f_u/∂u = -(w+1) + 2uv
    a[1] = uu;                // ∂f_u/∂v = u^2
    a[2] = -u;                // ∂f_u/∂w = -u
    a[3] = w - uv2;           // ∂f_v/∂u = w - 2uv
    a[4] = -uu;               // ∂f_v/∂v = -u^2
    a[5] = u;                 // ∂f_v/∂w = u
    a[6] = -w;                // ∂f_w/∂u = -w
    a[7] = 0.0;               // ∂f_w/∂v = 0
    a[8] = -inv_eps - u;      // ∂f_w/∂w = -1/eps - u
  }
}

// O9 advection f_E, first-order upwind for c > 0 (DESIGN R20),
// periodic.  Global grid nx × ny × nz cells (1D: ny = nz = 1),
// index ((k ny + j) nx + i)·3 + s.  Per axis: term = RN(kappa·RN(q_prev - q)),
// kappa = RN(c/Δ) precomputed by the caller.  Sum order: x, then + y, then
// + z (DESIGN R19).  Axes of extent 1 contribute nothing (1D / 2D).
void oracle_advection(int64_t nx, int64_t ny, int64_t nz, double kx, double ky,
                      double kz, const double* y, double* f) {
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        int64_t c = (k * ny + j) * nx + i;
        int64_t im = (i == 0 ? nx - 1 : i - 1);
        int64_t jm = (j == 0 ? ny - 1 : j - 1);
        int64_t km = (k == 0 ? nz - 1 : k - 1);
        int64_t cx = (k * ny + j) * nx + im;
        int64_t cy = (k * ny + jm) * nx + i;
        int64_t cz = (km * ny + j) * nx + i;
        for (int s = 0; s < 3; ++s) {
          double q = y[3 * c + s];
          double d = y[3 * cx + s] - q;
          double acc = kx * d;
          if (ny > 1) {
            double dy = y[3 * cy + s] - q;
            double ty = ky * dy;
            acc = acc + ty;
          }
          if (nz > 1) {
            double dz = y[3 * cz + s] - q;
            double tz = kz * dz;
            acc = acc + tz;
          }
          f[3 * c + s] = acc;
        }
      }
}

// O10 initial condition: p = α exp(-r²/(2σ²)), μ = L/2, σ = L/4
// per axis; u = A + p, v = B/A + p, w = 3 + p.  Coordinates x_i = i·Δ
// (uniform mesh).  r² = (x-μx)² [+ (y-μy)²] [+ (z-μz)²] in that order;
// 2σ² is per-axis-equal only for cubes, so the exponent is summed per axis:
// e = (x-μx)²/(2σx²) + (y-μy)²/(2σy²) + (z-μz)²/(2σz²).
void oracle_bruss_ic(int64_t nx, int64_t ny, int64_t nz, double Lx, double Ly,
                     double Lz, double A, double B, double alpha, double* y) {
  double dx = Lx / (double)nx, dy = Ly / (double)ny, dz = Lz / (double)nz;
  double mx = Lx / 2.0, my = Ly / 2.0, mz = Lz / 2.0;
  double sx = Lx / 4.0, sy = Ly / 4.0, sz = Lz / 4.0;
  double tx = 2.0 * (sx * sx), ty = 2.0 * (sy * sy), tz = 2.0 * (sz * sz);
  double BA = B / A;
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        double xe = (double)i * dx - mx;
        double e = (xe * xe) / tx;
        if (ny > 1) {
          double ye = (double)j * dy - my;
          e = e + (ye * ye) / ty;
        }
        if (nz > 1) {
          double ze = (double)k * dz - mz;
          e = e + (ze * ze) / tz;
        }
        double p = alpha * std::exp(-e);
        int64_t c = (k * ny + j) * nx + i;
        y[3 * c] = A + p;
        y[3 * c + 1] = BA + p;
        y[3 * c + 2] = 3.0 + p;
      }
}

// ---------------------------------------------------------------------------
// O11–O13: fixed-step IMEX-BDF (SBDF1 start, then SBDF2) with modified Newton
// on the implicit reaction (P:384-385 IMEX split: advection explicit, stiff
// reaction implicit; P:388-390 per-cell Newton with block solves; DESIGN
// R14/R15).  Steps:
//   f_E,n = advection(y_n)
//   n = 0:  d = 1·y_0 + h·f_E,0                       γ = h
//   n ≥ 1:  d = 4/3 y_n − 1/3 y_{n−1} + 4h/3 f_E,n − 2h/3 f_E,n−1   γ = 2h/3
//   ewt = 1/(rtol |y_n| + atol)   (Abs → Scale → AddConst → Inv)
//   z = y_n;  M = I − γ J(z)  (Jacobian, ScaleAddI(−γ)), LU factor
//   iterate: r = d + γ f_I(z) − z ; δ = M⁻¹ r ; z = z + δ ; ν = WRMS(δ, ewt)
//   y_{n+1} = z
// Problem kinds: 0 = Brusselator (reaction O8/O5, advection O9);
//                1 = linear test y' = λ_E y + λ_I y (f_E = λ_E y, f_I = λ_I y,
//                    J = λ_I I per 3×3 block).
// newton_mode: 0 fixed-K (exactly K iterations), 1 tolerance (stop when
// ν ≤ tol_nl, fail after K), 2 full convergence (iterate until
// ‖δ‖∞ ≤ 4u‖z‖∞ or 50 iterations; certifies K).
// ---------------------------------------------------------------------------

struct OracleSbdfParams {
  int32_t kind;           // 0 brusselator, 1 linear test
  int32_t newton_mode;    // 0 fixed-K, 1 tol, 2 full convergence
  int32_t K;
  int32_t reaction_only;  // 1: f_E = 0
  int64_t nx, ny, nz;     // global grid
  double kx, ky, kz;      // kappa per axis = c/Δ (RN)
  double A, B, eps;
  double lam_E, lam_I;
  double h, rtol, atol, tol_nl;
  int32_t linsol;         // 0: block LU solve (task-local); 2: block inverse by
                          // symbolic Gauss-Jordan; 1: GMRES, block-LU
                          //    preconditioner (the paper's global Newton)
  int32_t maxl;           // GMRES Krylov dimension
  double lin_tol;         // GMRES relative residual tolerance
};

int oracle_gmres(int64_t G, int m, const double* A, const double* PLU, const int32_t* Ppiv,
                 const double* b, double* x, int maxl, double tol, double* res);

struct OracleSbdfStats {
  int64_t steps;
  int64_t newton_iters;
  int64_t setups;
  int64_t solves;
  int64_t fails;          // tolerance-mode failures (recoverable)
  int64_t singular;       // 1 + first singular block at the first failure
  double last_nu;
  int64_t lin_iters;      // GMRES Arnoldi steps (linsol = 1)
};

static void rhs_explicit(const OracleSbdfParams* P, int64_t n, const double* y,
                         double* fE) {
  if (P->reaction_only) {
    for (int64_t i = 0; i < n; ++i) fE[i] = 0.0;
    return;
  }
  if (P->kind == 0)
    oracle_advection(P->nx, P->ny, P->nz, P->kx, P->ky, P->kz, y, fE);
  else
    oracle_scale(n, P->lam_E, y, fE);
}

static void rhs_implicit(const OracleSbdfParams* P, int64_t G, const double* y,
                         double* fI) {
  if (P->kind == 0)
    oracle_bruss_reaction(G, y, P->A, P->B, P->eps, fI);
  else
    oracle_scale(3 * G, P->lam_I, y, fI);
}

static void jac_implicit(const OracleSbdfParams* P, int64_t G, const double* y,
                         double* J) {
  if (P->kind == 0) {
    oracle_bruss_jacobian(G, y, P->eps, J);
  } else {
    for (int64_t g = 0; g < G; ++g)
      for (int e = 0; e < 9; ++e)
        J[9 * g + e] = (e % 4 == 0) ? P->lam_I : 0.0;
  }
}

// Evolves y (in/out, 3G values) by nsteps fixed steps.  ylog (optional,
// may be NULL) receives y after every log_every steps (log_every>0).
// Returns 0, or 1 on a recoverable failure (tolerance mode non-convergence
// or singular block), stopping at that step.
int oracle_sbdf_integrate(const OracleSbdfParams* P, double* y, int64_t nsteps,
                          OracleSbdfStats* st, double* ylog,
                          int64_t log_every) {
  int64_t G = P->nx * P->ny * P->nz;
  int64_t n = 3 * G;
  std::vector<double> yprev(n), fE(n), fEprev(n), d(n), ewt(n), z(n), fI(n),
      r(n), delta(n), M(9 * G), Mop(9 * G), tmp(n);
  std::vector<int32_t> piv(3 * G);
  std::memset(st, 0, sizeof(*st));
  int64_t nlog = 0;
  for (int64_t step = 0; step < nsteps; ++step) {
    rhs_explicit(P, n, y, fE.data());
    double gamma;
    if (step == 0) {
      oracle_linear_sum(n, 1.0, y, P->h, fE.data(), d.data());
      gamma = P->h;
    } else {
      // SBDF2 (P:384-385 IMEX split; R14 coefficients), d = 4/3 y_n - 1/3 y_{n-1}
      // + 4h/3 f_E,n - 2h/3 f_E,n-1, as one LinearCombination with the
      // history terms first (R28: the paper fixes no summation order)
      double c[4] = {-1.0 / 3.0, -((2.0 * P->h) / 3.0), 4.0 / 3.0,
                     (4.0 * P->h) / 3.0};
      const double* X[4] = {yprev.data(), fEprev.data(), y, fE.data()};
      oracle_linear_combination(4, c, X, n, d.data());
      gamma = (2.0 * P->h) / 3.0;
    }
    // ewt = 1/(rtol|y_n| + atol)
    oracle_abs(n, y, tmp.data());
    oracle_scale(n, P->rtol, tmp.data(), tmp.data());
    oracle_add_const(n, tmp.data(), P->atol, tmp.data());
    if (!(oracle_min(n, tmp.data()) > 0.0)) return 1;
    oracle_inv(n, tmp.data(), ewt.data());
    // predictor and Newton matrix at the predictor (modified Newton)
    std::memcpy(z.data(), y, n * sizeof(double));
    jac_implicit(P, G, z.data(), M.data());
    oracle_scale_add_identity(G, 3, -gamma, M.data());
    if (P->linsol == 1) Mop = M;            // the operator; M becomes its LU
    int64_t sing = P->linsol == 2 ? oracle_gj_inverse(G, 3, M.data(), Mop.data())
                                  : oracle_lu_factor(G, 3, M.data(), piv.data());
    st->setups++;
    if (sing) { st->singular = sing; st->fails++; return 1; }
    int maxit = (P->newton_mode == 2) ? 50 : P->K;
    bool converged = (P->newton_mode == 0);
    for (int it = 0; it < maxit; ++it) {
      rhs_implicit(P, G, z.data(), fI.data());
      double c3[3] = {1.0, gamma, -1.0};
      const double* X3[3] = {d.data(), fI.data(), z.data()};
      oracle_linear_combination(3, c3, X3, n, r.data());
      if (P->linsol == 1) {
        double res = 0.0;
        st->lin_iters += oracle_gmres(G, 3, Mop.data(), M.data(), piv.data(), r.data(),
                                      delta.data(), P->maxl, P->lin_tol, &res);
      } else if (P->linsol == 2) {
        oracle_gj_apply(G, 3, Mop.data(), r.data(), delta.data());
      } else {
        oracle_lu_solve(G, 3, M.data(), piv.data(), r.data(), delta.data());
      }
      st->solves++;
      oracle_linear_sum(n, 1.0, z.data(), 1.0, delta.data(), z.data());
      double nu = oracle_wrms(n, delta.data(), ewt.data());
      st->newton_iters++;
      st->last_nu = nu;
      if (P->newton_mode == 1 && nu <= P->tol_nl) { converged = true; break; }
      if (P->newton_mode == 2) {
        double dm = oracle_max_norm(n, delta.data());
        double zm = oracle_max_norm(n, z.data());
        if (dm <= 4.0 * 2.220446049250313e-16 * zm) { converged = true; break; }
      }
    }
    if (!converged) { st->fails++; return 1; }
    std::memcpy(yprev.data(), y, n * sizeof(double));
    std::memcpy(fEprev.data(), fE.data(), n * sizeof(double));
    std::memcpy(y, z.data(), n * sizeof(double));
    st->steps++;
    if (ylog && log_every > 0 && (step + 1) % log_every == 0) {
      std::memcpy(ylog + nlog * n, y, n * sizeof(double));
      ++nlog;
    }
  }
  return 0;
}

// ---------------------------------------------------------------------------
// GMRES (the SPGMR Krylov solver of P:299 §5, used by the paper's "global"
// Newton configuration with the block solve as preconditioner, §7).
// Right-preconditioned GMRES(maxl) without restarts, x0 = 0:
//   β = ‖b‖₂, V₀ = b/β
//   for j = 0..maxl-1:
//     w = A P⁻¹ V_j
//     h_ij = w·V_i (i ≤ j)                  — classical Gram–Schmidt: all
//     w = w − Σ_i h_ij V_i                    inner products from the same w
//     h_{j+1,j} = ‖w‖₂, V_{j+1} = w / h_{j+1,j}
//     Givens rotations on column j; |g_{j+1}| = residual norm
//     stop if |g_{j+1}| ≤ tol·β (or h_{j+1,j} == 0)
//   y = H⁻¹ g (back substitution), x = P⁻¹ Σ_i y_i V_i
// A: G blocks of m×m (row-major), PLU/Ppiv: LU factors + pivots of the
// block preconditioner (oracle_lu_factor format), or NULL for P = I.
// Returns the number of Arnoldi steps; *res = final |g_{j+1}|.
static void block_solve_or_copy(int64_t G, int m, const double* LU, const int32_t* piv,
                                const double* v, double* out) {
  if (LU)
    oracle_lu_solve(G, m, LU, piv, v, out);
  else
    std::memcpy(out, v, sizeof(double) * G * m);
}

int oracle_gmres(int64_t G, int m, const double* A, const double* PLU, const int32_t* Ppiv,
                 const double* b, double* x, int maxl, double tol, double* res) {
  const int64_t n = G * m;
  std::vector<std::vector<double>> V(maxl + 1, std::vector<double>(n));
  std::vector<double> H((maxl + 1) * maxl, 0.0), g(maxl + 1, 0.0), cs(maxl), sn(maxl);
  std::vector<double> z(n), w(n);
  double beta = std::sqrt(oracle_dot(n, b, b));
  if (beta == 0.0) {
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    *res = 0.0;
    return 0;
  }
  oracle_scale(n, 1.0 / beta, b, V[0].data());
  g[0] = beta;
  int j = 0, steps = 0;
  for (; j < maxl; ++j) {
    block_solve_or_copy(G, m, PLU, Ppiv, V[j].data(), z.data());
    oracle_block_matvec(G, m, A, z.data(), w.data());
    for (int i = 0; i <= j; ++i) H[i * maxl + j] = oracle_dot(n, w.data(), V[i].data());
    for (int i = 0; i <= j; ++i) {
      double c = -H[i * maxl + j];
      for (int64_t k = 0; k < n; ++k) {
        double t = c * V[i][k];
        w[k] = w[k] + t;
      }
    }
    double hn = std::sqrt(oracle_dot(n, w.data(), w.data()));
    H[(j + 1) * maxl + j] = hn;
    if (hn != 0.0) oracle_scale(n, 1.0 / hn, w.data(), V[j + 1].data());
    for (int i = 0; i < j; ++i) {            // previous rotations on column j
      double a = H[i * maxl + j], c = H[(i + 1) * maxl + j];
      H[i * maxl + j] = cs[i] * a + sn[i] * c;
      H[(i + 1) * maxl + j] = -sn[i] * a + cs[i] * c;
    }
    double a = H[j * maxl + j], c = H[(j + 1) * maxl + j];
    double r = std::hypot(a, c);
    cs[j] = a / r;
    sn[j] = c / r;
    H[j * maxl + j] = r;
    H[(j + 1) * maxl + j] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    steps = j + 1;
    if (std::fabs(g[j + 1]) <= tol * beta || hn == 0.0) break;
  }
  std::vector<double> y(steps);
  for (int i = steps - 1; i >= 0; --i) {
    double s = g[i];
    for (int k = i + 1; k < steps; ++k) s -= H[i * maxl + k] * y[k];
    y[i] = s / H[i * maxl + i];
  }
  for (int64_t k = 0; k < n; ++k) {
    double s = 0.0;
    for (int i = 0; i < steps; ++i) s += y[i] * V[i][k];
    w[k] = s;
  }
  block_solve_or_copy(G, m, PLU, Ppiv, w.data(), x);
  *res = std::fabs(g[steps]);
  return steps;
}

// ---------------------------------------------------------------------------
// Adaptive IMEX additive Runge–Kutta — the paper's integrator (ARKODE IMEX,
// advection explicit, reaction implicit; temporal error control
// through global reductions and step recomputation with a smaller h when a
// nonlinear solve fails).  Tableau: ARK3(2)4L[2]SA of Kennedy and
// Carpenter (the paper names no tableau; SPEC S:418 picks this one; DESIGN
// R26).  Stages i = 1..4 (a^I_11 = 0: the first stage is explicit):
//   Z_i = y_n + h Σ_{j<i} (aE_ij FE_j + aI_ij FI_j) + h γ f_I(Z_i)
//   FE_i = f_E(Z_i), FI_i = f_I(Z_i)
//   y_{n+1} = y_n + h Σ_i b_i (FE_i + FI_i)
//   e = h Σ_i (b_i − d_i)(FE_i + FI_i),  dsm = WRMS(e, ewt(y_n))
// Stage solve: modified Newton, M = I − hγ J(Z_{i−1}) (predictor: previous
// stage), r = rhs + hγ f_I(Z) − Z, δ = M⁻¹r, Z += δ, ν = WRMS(δ, ewt);
// converged when ν ≤ tol_nl, failure after maxnl iterations → the step is
// recomputed with h·0.25.  Step control (I-controller, DESIGN R26):
// accept if dsm ≤ 1; h ← h·min(5, max(0.2, 0.9·dsm^(−1/3))) (rejection: max
// factor 1).  The Newton matrix of a stage is the Jacobian of the reaction
// only, exactly block diagonal.
// ---------------------------------------------------------------------------

struct OracleArkParams {
  OracleSbdfParams prob;  // kind, grid, kappas, A/B/eps, lambdas, rtol/atol, tol_nl
  double h0;              // initial step
  double t_end;           // integrate [0, t_end]
  int32_t maxnl;          // Newton iterations per stage
  int32_t max_steps;      // attempts (accepted + rejected) limit
  int32_t fixed;          // 1: constant h, every step accepted (order pins)
  int32_t pad_;
};

struct OracleArkStats {
  int64_t accepted, rejected_err, rejected_nl, newton_iters, setups;
  double t, h_last;
};

static const double ARK_G = 1767732205903.0 / 4055673282236.0;
static const double ARK_C[4] = {0.0, 1767732205903.0 / 2027836641118.0, 3.0 / 5.0, 1.0};
static const double ARK_AE[4][4] = {
    {0, 0, 0, 0},
    {1767732205903.0 / 2027836641118.0, 0, 0, 0},
    {5535828885825.0 / 10492691773637.0, 788022342437.0 / 10882634858940.0, 0, 0},
    {6485989280629.0 / 16251701735622.0, -4246266847089.0 / 9704473918619.0,
     10755448449292.0 / 10357097424841.0, 0}};
static const double ARK_AI[4][4] = {
    {0, 0, 0, 0},
    {1767732205903.0 / 4055673282236.0, 1767732205903.0 / 4055673282236.0, 0, 0},
    {2746238789719.0 / 10658868560708.0, -640167445237.0 / 6845629431997.0,
     1767732205903.0 / 4055673282236.0, 0},
    {1471266399579.0 / 7840856788654.0, -4482444167858.0 / 7529755066697.0,
     11266239266428.0 / 11593286722821.0, 1767732205903.0 / 4055673282236.0}};
static const double ARK_B[4] = {1471266399579.0 / 7840856788654.0, -4482444167858.0 / 7529755066697.0,
                                11266239266428.0 / 11593286722821.0, 1767732205903.0 / 4055673282236.0};
static const double ARK_D[4] = {2756255671327.0 / 12835298489170.0, -10771552573575.0 / 22201958757719.0,
                                9247589265047.0 / 10645013368117.0, 2193209047091.0 / 5459859503100.0};

// the tableau as doubles (for the order-condition pins)
void oracle_ark_tableau(double* AE16, double* AI16, double* b4, double* d4, double* c4) {
  for (int i = 0; i < 4; ++i) {
    b4[i] = ARK_B[i];
    d4[i] = ARK_D[i];
    c4[i] = ARK_C[i];
    for (int j = 0; j < 4; ++j) {
      AE16[4 * i + j] = ARK_AE[i][j];
      AI16[4 * i + j] = ARK_AI[i][j];
    }
  }
}

// Returns 0 (reached t_end), 1 (max_steps exhausted) or 2 (h underflow).
int oracle_ark_integrate(const OracleArkParams* AP, double* y, OracleArkStats* st) {
  const OracleSbdfParams* P = &AP->prob;
  int64_t G = P->nx * P->ny * P->nz;
  int64_t n = 3 * G;
  std::vector<double> ewt(n), tmp(n), rhs(n), Z(n), r(n), delta(n), ynew(n), err(n), fI(n),
      M(9 * G);
  std::vector<int32_t> piv(3 * G);
  std::vector<std::vector<double>> FE(4, std::vector<double>(n)), FI(4, std::vector<double>(n));
  std::memset(st, 0, sizeof(*st));
  double t = 0.0, h = AP->h0;
  int attempts = 0;
  // done when the remaining interval is below 1e-12·max(1, |t_end|)
  // (accumulated rounding of t; DESIGN R26)
  while (AP->t_end - t > 1e-12 * std::fmax(1.0, std::fabs(AP->t_end))) {
    if (attempts++ >= AP->max_steps) { st->t = t; st->h_last = h; return 1; }
    // a step shortened to land on t_end does not shrink the controller's
    // next proposal (DESIGN R26): the unclipped h is kept for after it
    const double h_unclipped = h;
    const bool clipped = t + h > AP->t_end;
    if (clipped) h = AP->t_end - t;
    if (h < 1e-14 * (1.0 + t)) { st->t = t; st->h_last = h; return 2; }
    // ewt from y_n
    oracle_abs(n, y, tmp.data());
    oracle_scale(n, P->rtol, tmp.data(), tmp.data());
    oracle_add_const(n, tmp.data(), P->atol, tmp.data());
    oracle_inv(n, tmp.data(), ewt.data());
    const double hg = h * ARK_G;
    bool nl_fail = false;
    for (int i = 0; i < 4 && !nl_fail; ++i) {
      if (i == 0) {
        std::memcpy(Z.data(), y, n * sizeof(double));
      } else {
        // rhs = y_n + h Σ_{j<i} (aE_ij FE_j + aI_ij FI_j)
        std::vector<double> c;
        std::vector<const double*> X;
        c.push_back(1.0);
        X.push_back(y);
        for (int j = 0; j < i; ++j) {
          c.push_back(h * ARK_AE[i][j]); X.push_back(FE[j].data());
          c.push_back(h * ARK_AI[i][j]); X.push_back(FI[j].data());
        }
        oracle_linear_combination((int)c.size(), c.data(), X.data(), n, rhs.data());
        // modified Newton from the previous stage value (Z holds Z_{i-1})
        jac_implicit(P, G, Z.data(), M.data());
        oracle_scale_add_identity(G, 3, -hg, M.data());
        st->setups++;
        if (oracle_lu_factor(G, 3, M.data(), piv.data())) { nl_fail = true; break; }
        bool conv = false;
        for (int it = 0; it < AP->maxnl; ++it) {
          rhs_implicit(P, G, Z.data(), fI.data());
          double c3[3] = {1.0, hg, -1.0};
          const double* X3[3] = {rhs.data(), fI.data(), Z.data()};
          oracle_linear_combination(3, c3, X3, n, r.data());
          oracle_lu_solve(G, 3, M.data(), piv.data(), r.data(), delta.data());
          oracle_linear_sum(n, 1.0, Z.data(), 1.0, delta.data(), Z.data());
          st->newton_iters++;
          if (oracle_wrms(n, delta.data(), ewt.data()) <= P->tol_nl) { conv = true; break; }
        }
        if (!conv) { nl_fail = true; break; }
      }
      rhs_explicit(P, n, Z.data(), FE[i].data());
      rhs_implicit(P, G, Z.data(), FI[i].data());
    }
    if (nl_fail) {               // recompute the step with a smaller h
      st->rejected_nl++;
      h *= 0.25;
      continue;
    }
    // y_{n+1} and the embedded error
    {
      std::vector<double> c, ce;
      std::vector<const double*> X, Xe;
      c.push_back(1.0);
      X.push_back(y);
      for (int i = 0; i < 4; ++i) {
        c.push_back(h * ARK_B[i]); X.push_back(FE[i].data());
        c.push_back(h * ARK_B[i]); X.push_back(FI[i].data());
        double be = h * (ARK_B[i] - ARK_D[i]);
        ce.push_back(be); Xe.push_back(FE[i].data());
        ce.push_back(be); Xe.push_back(FI[i].data());
      }
      oracle_linear_combination((int)c.size(), c.data(), X.data(), n, ynew.data());
      oracle_linear_combination((int)ce.size(), ce.data(), Xe.data(), n, err.data());
    }
    double dsm = oracle_wrms(n, err.data(), ewt.data());
    double fac = dsm > 0.0 ? 0.9 * std::pow(dsm, -1.0 / 3.0) : 5.0;
    if (AP->fixed) { dsm = 0.0; fac = 1.0; }
    if (dsm <= 1.0) {
      std::memcpy(y, ynew.data(), n * sizeof(double));
      t += h;
      st->accepted++;
      h *= std::fmin(5.0, std::fmax(0.2, fac));
      if (clipped) h = std::fmax(h, h_unclipped);
    } else {
      st->rejected_err++;
      h *= std::fmin(1.0, std::fmax(0.2, fac));
    }
  }
  st->t = t;
  st->h_last = h;
  return 0;
}

int oracle_abi_version(void) { return 1; }

}  // extern "C"

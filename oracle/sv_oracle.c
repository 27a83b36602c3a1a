/*
 * sv_oracle.c -- O1, the CPU oracle for the simulation result.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2408_09055_b200/), and never calls it.
 *
 * What it computes: the plain definition the method reaches exactly,
 *     |psi> = U_m ... U_1 |psi_0>,
 * applying the gates one at a time (Eq. 2, generalised
 * to k-qubit gates as in SPEC S:L391-394).  Staging, kernelization, insular
 * specialisation and remapping are exact rewrites of this product
 * ("work for arbitrary input states"), so the oracle needs none of them.
 *
 * Arithmetic: complex128 (P:L1964 footnote: "2 double-precision floating-point
 * numbers"), straight loops, no fusion, no reordering.
 *
 * Gate matrices: textbook / OpenQASM definitions, written out here (SURVEY
 * §8c O1).  Matrix index convention: operand qubits[0] is the least significant
 * bit of the row/column index.  Qubit q is bit q of the amplitude
 * index (pairs (f(i), f(i)+2^q)).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* Kind codes of the oracle's own table (mapped from kind names in oracle/sim.py). */
enum {
  O_H = 0, O_X, O_Y, O_Z, O_S, O_SDG, O_T, O_TDG, O_RX, O_RY, O_RZ, O_P, O_U3,
  O_CX, O_CZ, O_CP, O_CCX, O_SWAP, O_CU, O_NKINDS
};

static int arity(int kind) {
  if (kind <= O_U3) return 1;
  if (kind == O_CCX) return 3;
  return 2;
}

/* Fill U (dim x dim, row-major) for the gate.  Returns dim or -1. */
int oracle_gate_matrix(int kind, const double *p, double *out_re, double *out_im) {
  cplx U[64];
  int k = (kind >= 0 && kind < O_NKINDS) ? arity(kind) : -1;
  if (k < 0) return -1;
  int d = 1 << k;
  for (int i = 0; i < d * d; i++) U[i] = 0;
  const double r2 = 1.0 / sqrt(2.0);
  double c, s;
  switch (kind) {
    case O_H: U[0] = r2; U[1] = r2; U[2] = r2; U[3] = -r2; break;
    case O_X: U[1] = 1; U[2] = 1; break;
    case O_Y: U[1] = -I; U[2] = I; break;
    case O_Z: U[0] = 1; U[3] = -1; break;
    case O_S: U[0] = 1; U[3] = I; break;
    case O_SDG: U[0] = 1; U[3] = -I; break;
    case O_T: U[0] = 1; U[3] = cexp(I * M_PI / 4); break;
    case O_TDG: U[0] = 1; U[3] = cexp(-I * M_PI / 4); break;
    case O_RX: /* [[c, -i s], [-i s, c]] */
      c = cos(p[0] / 2); s = sin(p[0] / 2);
      U[0] = c; U[1] = -I * s; U[2] = -I * s; U[3] = c; break;
    case O_RY: /* [[c, -s], [s, c]] */
      c = cos(p[0] / 2); s = sin(p[0] / 2);
      U[0] = c; U[1] = -s; U[2] = s; U[3] = c; break;
    case O_RZ: /* diag(e^{-i t/2}, e^{i t/2}) */
      U[0] = cexp(-I * p[0] / 2); U[3] = cexp(I * p[0] / 2); break;
    case O_P: U[0] = 1; U[3] = cexp(I * p[0]); break;
    case O_U3: /* [[c, -e^{i lam} s], [e^{i phi} s, e^{i(phi+lam)} c]] */
      c = cos(p[0] / 2); s = sin(p[0] / 2);
      U[0] = c; U[1] = -cexp(I * p[2]) * s;
      U[2] = cexp(I * p[1]) * s; U[3] = cexp(I * (p[1] + p[2])) * c; break;
    case O_CX: /* control = qubits[0] (index bit 0), target = qubits[1] (bit 1) */
      U[0 * 4 + 0] = 1; U[2 * 4 + 2] = 1; U[1 * 4 + 3] = 1; U[3 * 4 + 1] = 1; break;
    case O_CZ: U[0] = 1; U[5] = 1; U[10] = 1; U[15] = -1; break;
    case O_CP: U[0] = 1; U[5] = 1; U[10] = 1; U[15] = cexp(I * p[0]); break;
    case O_SWAP: U[0] = 1; U[1 * 4 + 2] = 1; U[2 * 4 + 1] = 1; U[15] = 1; break;
    case O_CU: { /* OpenQASM 3 cu(theta, phi, lambda, gamma): control=bit0 */
      cplx u[4];
      c = cos(p[0] / 2); s = sin(p[0] / 2);
      u[0] = c; u[1] = -cexp(I * p[2]) * s;
      u[2] = cexp(I * p[1]) * s; u[3] = cexp(I * (p[1] + p[2])) * c;
      U[0] = 1; U[2 * 4 + 2] = 1;
      for (int r = 0; r < 2; r++)
        for (int cc = 0; cc < 2; cc++)
          U[(1 + 2 * r) * 4 + (1 + 2 * cc)] = cexp(I * p[3]) * u[r * 2 + cc];
      break;
    }
    case O_CCX: /* controls bits 0,1; target bit 2: index 3 <-> 7 */
      for (int i = 0; i < 8; i++) if (i != 3 && i != 7) U[i * 8 + i] = 1;
      U[3 * 8 + 7] = 1; U[7 * 8 + 3] = 1; break;
    default: return -1;
  }
  for (int i = 0; i < d * d; i++) { out_re[i] = creal(U[i]); out_im[i] = cimag(U[i]); }
  return d;
}

/*
 * Apply one k-qubit gate (qubits q[0..k-1], q[0] = matrix LSB) to the state
 * psi (2^n amplitudes, interleaved re,im).  For every index i whose target
 * bits are all zero: gather v[c] = psi[i + sum_j c_j 2^{q_j}], w = U v,
 * scatter w back.  For k = 1 this is exactly Eq. 2.
 */
int oracle_apply_gate(double *psi, int n, int kind, const int *q, const double *p) {
  double ure[64], uim[64];
  int d = oracle_gate_matrix(kind, p, ure, uim);
  if (d < 0) return -1;
  int k = arity(kind);
  uint64_t mask = 0, off[8];
  for (int j = 0; j < k; j++) {
    if (q[j] < 0 || q[j] >= n) return -2;
    if (mask & (1ULL << q[j])) return -3;
    mask |= 1ULL << q[j];
  }
  for (int c = 0; c < d; c++) {
    off[c] = 0;
    for (int j = 0; j < k; j++) if ((c >> j) & 1) off[c] |= 1ULL << q[j];
  }
  cplx *s = (cplx *)psi;
  const uint64_t N = 1ULL << n;
  /* The iterations touch disjoint amplitude groups, so the OpenMP build
   * (liboracle_omp.so, -fopenmp) splits them over the host cores; every
   * amplitude gets the same arithmetic in the same order as in the 1-thread
   * build (bit-identical results). */
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < N; i++) {
    cplx v[8], w[8];
    if (i & mask) continue;
    for (int c = 0; c < d; c++) v[c] = s[i + off[c]];
    for (int r = 0; r < d; r++) {
      cplx acc = 0;
      for (int c = 0; c < d; c++) acc += (ure[r * d + c] + I * uim[r * d + c]) * v[c];
      w[r] = acc;
    }
    for (int c = 0; c < d; c++) s[i + off[c]] = w[c];
  }
  return 0;
}

/*
 * Simulate m gates on the state psi in place.  kinds[m], qubits[m*3],
 * params[m*4].  If init_zero, psi is first set to |0...0>.
 */
int oracle_simulate(double *psi, int n, int m, const int *kinds, const int *qubits,
                    const double *params, int init_zero) {
  if (n < 1 || n > 40) return -4;
  if (init_zero) {
    memset(psi, 0, sizeof(double) * 2 * (1ULL << n));
    psi[0] = 1.0;
  }
  for (int g = 0; g < m; g++) {
    int rc = oracle_apply_gate(psi, n, kinds[g], qubits + 3 * g, params + 4 * g);
    if (rc) return rc;
  }
  return 0;
}

/* Threads the OpenMP build uses (1 in the plain build). */
#ifdef _OPENMP
#include <omp.h>
int oracle_threads(void) { return omp_get_max_threads(); }
#else
int oracle_threads(void) { return 1; }
#endif

/* Squared norm sum |alpha_i|^2, for the norm-preservation pin. */
double oracle_norm2(const double *psi, int n) {
  double acc = 0;
  const uint64_t N = 1ULL << n;
  for (uint64_t i = 0; i < 2 * N; i++) acc += psi[i] * psi[i];
  return acc;
}

/*
 * CPU ORACLE KERNELS - TEST INFRASTRUCTURE / CPU BASELINE ONLY.
 *
 * Plain-C restatement of the reference's L1 kernels (parpf/accel.py), the
 * role the reference's numba twins play: lorenz_euler_block (accel.py:82-96),
 * fhn_euler_block (accel.py:110-129, general rectangular form, i.e. the
 * numpy twin's semantics) and resample_indices (accel.py:186-197).
 * Compiled with -ffp-contract=off so every operation rounds once, in the
 * reference's order: results are bit-identical to the reference's numpy and
 * numba twins (tests/test_oracle_golden.py, test_oracle_ckernels).
 * Used by oracle/ckernels.py for the bench's CPU baseline; never by the
 * product package.
 */
#include <math.h>
#include <stdint.h>

void orc_lorenz_euler_block(const double *states, const double *noise, int64_t n,
                            int64_t n_sub, double dt, double s, double r, double b,
                            double *out) {
  const double sq = sqrt(dt);
  const double dts = dt * s;
  for (int64_t i = 0; i < 3 * n; ++i) out[i] = states[i];
  for (int64_t k = 0; k < n_sub; ++k) {
    const double *z = noise + k * n * 3;
    for (int64_t i = 0; i < n; ++i) {
      const double x1 = out[3 * i], x2 = out[3 * i + 1], x3 = out[3 * i + 2];
      out[3 * i] = x1 - dts * (x1 - x2) + sq * z[3 * i];
      out[3 * i + 1] = x2 + dt * (r * x1 - x2 - x1 * x3) + sq * z[3 * i + 1];
      out[3 * i + 2] = x3 + dt * (x1 * x2 - b * x3) + sq * z[3 * i + 2];
    }
  }
}

void orc_fhn_euler_block(const double *U, const double *V, const double *drive,
                         const double *noise, int64_t n, int64_t J1, int64_t J2, double dt,
                         double coupling, const double *cubic, const double *beta,
                         double sig_sqdt, double *u_new, double *v_new) {
  const double a3 = cubic[0], a2 = cubic[1], a1 = cubic[2], a0 = cubic[3];
  const double b0 = beta[0], b1 = beta[1], b2 = beta[2];
  const int64_t plane = J1 * J2;
  for (int64_t p = 0; p < n; ++p) {
    const double *Up = U + p * plane;
    for (int64_t i = 0; i < J1; ++i)
      for (int64_t j = 0; j < J2; ++j) {
        const int64_t g = p * plane + i * J2 + j;
        double nb = 0.0;
        if (i > 0) nb += Up[(i - 1) * J2 + j];
        if (i < J1 - 1) nb += Up[(i + 1) * J2 + j];
        if (j > 0) nb += Up[i * J2 + j - 1];
        if (j < J2 - 1) nb += Up[i * J2 + j + 1];
        const double u = U[g], v = V[g];
        const double p3 = ((a3 * u + a2) * u + a1) * u + a0;
        u_new[g] = u + dt * (p3 - v) + dt * (coupling * nb + drive[g]) + sig_sqdt * noise[g];
        v_new[g] = v + dt * (b0 * u + b1 * v + b2);
      }
  }
}

void orc_resample_indices(const double *cum, int64_t n, const double *u, int64_t m,
                          int64_t *idx) {
  int64_t k = 0;
  for (int64_t j = 0; j < m; ++j) {
    while (k < n - 1 && cum[k] < u[j]) ++k;
    idx[j] = k;
  }
}

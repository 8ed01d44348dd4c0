/* Covariance tiles by direct differences -- the oracle's `cov` (oracle/covariance.py)
 * written out in plain C so that full-size references (a 262144 x 262144 root block, C a on
 * sampled rows of n = 2^20 points) finish in minutes on the host.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no
 * code with paper_1701_00285_b200/csrc/.
 *
 * What it computes (same definitions as oracle/covariance.py):
 *   r_ij  = sqrt( sum_k (xa_ik - xb_jk)^2 )          direct differences, summed k = 0..d-1
 *                                                     in order; NOT the Gram identity
 *   phi   = Matern closed forms of the definition P:970 (reading R16), z = sqrt(2 nu) r / rho:
 *             nu = 1/2: exp(-z);  nu = 3/2: (1 + z) exp(-z);  nu = 5/2: (1 + z + z^2/3) exp(-z)
 *           Gaussian exp(-r^2 / rho^2) (reading R17, BASELINE binds rho^2, not 2 rho^2)
 *   C_ij  = sigma2 * phi(r_ij) + nugget * [ia_i == ib_j]   (reading R18)
 * Each entry is computed on its own; the OpenMP loop only distributes independent rows, so
 * the result does not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { MATERN_12 = 0, MATERN_32 = 1, MATERN_52 = 2, GAUSSIAN = 3 };

static double phi(double r, int family, double rho)
{
    double z;
    switch (family) {
    case MATERN_12:
        z = r / rho;
        return exp(-z);
    case MATERN_32:
        z = sqrt(3.0) * r / rho;
        return (1.0 + z) * exp(-z);
    case MATERN_52:
        z = sqrt(5.0) * r / rho;
        return (1.0 + z + z * z / 3.0) * exp(-z);
    case GAUSSIAN:
        return exp(-(r * r) / (rho * rho));
    default:
        return NAN;
    }
}

/* out[i * nb + j] = C(xa_i, xb_j), Xa na x d and Xb nb x d row-major, ia / ib the global
 * observation indices.  Returns 0, or -1 for an unknown family / allocation failure. */
int oracle_cov_tile(const double* Xa, const int64_t* ia, int64_t na, const double* Xb,
                    const int64_t* ib, int64_t nb, int32_t d, int32_t family, double rho,
                    double sigma2, double nugget, double* out)
{
    if (family < MATERN_12 || family > GAUSSIAN) return -1;
    /* Xb transposed (d x nb) so the loop over j is contiguous */
    double* XbT = (double*)malloc(sizeof(double) * (size_t)nb * (size_t)(d > 0 ? d : 1));
    if (!XbT) return -1;
    for (int64_t j = 0; j < nb; ++j)
        for (int32_t k = 0; k < d; ++k) XbT[(size_t)k * nb + j] = Xb[(size_t)j * d + k];

    /* rows in groups of 16, columns in panels of 512 (the panel of Xb^T stays in cache for
     * the group's rows); every entry is still summed over k = 0..d-1 in order */
    const int64_t NI = 16, NJ = 512;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i0 = 0; i0 < na; i0 += NI) {
        double acc[512];
        const int64_t i1 = i0 + NI < na ? i0 + NI : na;
        for (int64_t j0 = 0; j0 < nb; j0 += NJ) {
            const int64_t nj = j0 + NJ < nb ? NJ : nb - j0;
            for (int64_t i = i0; i < i1; ++i) {
                for (int64_t j = 0; j < nj; ++j) acc[j] = 0.0;
                for (int32_t k = 0; k < d; ++k) {       /* s_ij += (x_ik - y_jk)^2, k in order */
                    const double xik = Xa[(size_t)i * d + k];
                    const double* yk = XbT + (size_t)k * nb + j0;
                    for (int64_t j = 0; j < nj; ++j) {
                        const double t = xik - yk[j];
                        acc[j] += t * t;
                    }
                }
                double* row = out + (size_t)i * nb + j0;
                for (int64_t j = 0; j < nj; ++j) {
                    double c = sigma2 * phi(sqrt(acc[j]), family, rho);
                    if (nugget != 0.0 && ia[i] == ib[j0 + j]) c += nugget;
                    row[j] = c;
                }
            }
        }
    }
    free(XbT);
    return 0;
}

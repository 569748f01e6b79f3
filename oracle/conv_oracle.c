/*
 * conv_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously correct CPU oracle for the hot path of
 * arXiv 2212.00404 (direct valid-mode stride-1 convolution).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, table or helper with the
 * CUDA path under paper_2212_00404_b200/ and neither side includes the other.
 *
 * What it computes (§2.1 "The Convolution Models", Eq. 1):
 *
 *   O^m(x,y) = sum_{ch} sum_{i=0}^{K-1} sum_{j=0}^{K-1} I^ch(x+i, y+j) * F^{ch,m}(i,j),
 *   x in [0, Wx-K+1), y in [0, Wy-K+1), m in [1, M]
 *
 * with C = 1 giving the single-channel Eq. 2.  Readings taken
 * (SURVEY.md §8(c)):
 *   Q1  the filter row index r ("i" = row, outer) pairs with the
 *       feature-map row y, the column index c with x, i.e.
 *         O[m][y][x] = sum_{ch,r,c} I[ch][y+r][x+c] * F[m][ch][r][c]
 *       (cross-correlation, = torch.nn.functional.conv2d on NCHW/OIHW, N=1);
 *   Q2  no kernel flip;  Q3 all indices 0-based;
 *   Q5  layouts I[ch][y][x], O[m][y][x], x fastest, no padding;
 *   D3  multi-channel filter layout "along the dimension ch first, and then
 *       along the dimension m" = F[m][ch][r][c], offset
 *       (((m*C+ch)*K+r)*K+c).
 * Accumulation is in 64-bit reals, summed in the order
 * ch, r, c of Eq. 1's sums; the result is returned in double (no rounding).
 * Alongside O the oracle returns the magnitude plane
 *   A^m(x,y) = sum_{ch,r,c} |I[ch][y+r][x+c] * F[m][ch][r][c]|
 * which scales the per-output tolerance of north_star (tol * sum |I||F|).
 *
 * Parallelism: an OpenMP loop over m only; every output's summation order is
 * exactly the sequential one, so results are bit-identical for
 * any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

/* Returns 0 on success, 1 on a shape error (any dim < 1, K > min(Wx,Wy)). */
int oracle_conv(const float *I, int C, int Wx, int Wy,
                const float *F, int K, int M,
                double *O, double *A)
{
    if (C < 1 || Wx < 1 || Wy < 1 || K < 1 || M < 1) return 1;
    if (K > Wx || K > Wy) return 1;
    const int Wo = Wx - K + 1;           /* x in [0, Wx-K+1) */
    const int Ho = Wy - K + 1;           /* y in [0, Wy-K+1) */
    const int64_t plane_in = (int64_t)Wx * Wy;
    const int64_t plane_out = (int64_t)Wo * Ho;

    int m;
#pragma omp parallel for schedule(dynamic, 1)
    for (m = 0; m < M; ++m) {
        for (int y = 0; y < Ho; ++y) {
            for (int x = 0; x < Wo; ++x) {
                double s = 0.0, a = 0.0;
                for (int ch = 0; ch < C; ++ch) {              /* sum over ch  */
                    const float *Ic = I + (int64_t)ch * plane_in;
                    const float *Fmc = F + ((int64_t)m * C + ch) * K * K;
                    for (int r = 0; r < K; ++r) {             /* sum over i   */
                        for (int c = 0; c < K; ++c) {         /* sum over j   */
                            double p = (double)Ic[(int64_t)(y + r) * Wx + (x + c)]
                                     * (double)Fmc[r * K + c];
                            s += p;
                            a += fabs(p);
                        }
                    }
                }
                int64_t o = (int64_t)m * plane_out + (int64_t)y * Wo + x;
                O[o] = s;
                if (A) A[o] = a;
            }
        }
    }
    return 0;
}

/* Sampled variant for outputs at full BASELINE sizes: computes only the
 * outputs listed in idx (flat indices into O[m][y][x]); same arithmetic and
 * summation order as oracle_conv, one output at a time. */
int oracle_conv_sampled(const float *I, int C, int Wx, int Wy,
                        const float *F, int K, int M,
                        const int64_t *idx, int64_t n,
                        double *O, double *A)
{
    if (C < 1 || Wx < 1 || Wy < 1 || K < 1 || M < 1) return 1;
    if (K > Wx || K > Wy) return 1;
    const int Wo = Wx - K + 1;
    const int Ho = Wy - K + 1;
    const int64_t plane_in = (int64_t)Wx * Wy;
    const int64_t plane_out = (int64_t)Wo * Ho;
    int64_t t;
#pragma omp parallel for schedule(static)
    for (t = 0; t < n; ++t) {
        int64_t o = idx[t];
        int m = (int)(o / plane_out);
        int64_t rem = o % plane_out;
        int y = (int)(rem / Wo), x = (int)(rem % Wo);
        double s = 0.0, a = 0.0;
        if (m < M) {
            for (int ch = 0; ch < C; ++ch) {
                const float *Ic = I + (int64_t)ch * plane_in;
                const float *Fmc = F + ((int64_t)m * C + ch) * K * K;
                for (int r = 0; r < K; ++r)
                    for (int c = 0; c < K; ++c) {
                        double p = (double)Ic[(int64_t)(y + r) * Wx + (x + c)]
                                 * (double)Fmc[r * K + c];
                        s += p;
                        a += fabs(p);
                    }
            }
        }
        O[t] = s;
        if (A) A[t] = a;
    }
    return 0;
}

#ifdef _OPENMP
#include <omp.h>
#endif
/* Thread control for the timed CPU baseline; returns the count in effect. */
int oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

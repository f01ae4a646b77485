/* oracle/clawref_impl.h -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * Plain-C restatement of the reference's fused pencil sweep, instantiated
 * twice by clawref.c (T=float, T=double).  Nothing in the product links
 * this; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg load it.
 *
 * Every arithmetic expression keeps the reference's evaluation order and
 * is compiled with -ffp-contract=off, so results are IEEE-identical to the
 * numba kernel (which is itself bit-identical to its interpreted py_func,
 * pkg/tests/test_riemann.py:192-217).
 *
 * Sources restated (paths relative to /root/reference/pkg/src/clawtile):
 *   limiter_value        sweep.py:158-181
 *   sweep_tile           sweep.py:183-263
 *   _acoustics_scalar    riemann.py:116-133   (params [c, Z, T(0.5)/T(Z)])
 *   _shallow_water_scalar riemann.py:136-167  (params [g, 0.5])
 *   _advection_scalar    riemann.py:170-173   (params [u])
 *   vc_acoustics         builder extension; states
 *                        (p, u[, v[, w]], Z, c), zero waves on Z and c.
 */

#ifndef T
#error "define T before including clawref_impl.h"
#endif

#define CR_CAT2(a, b) a##b
#define CR_CAT(a, b) CR_CAT2(a, b)
#define CR_FN(name) CR_CAT(name, SUF)


/* sweep.py:158-181 */
static T CR_FN(limiter_value)(T theta, int kind)
{
    const T ZERO = (T)0.0, HALF = (T)0.5, ONE = (T)1.0, TWO = (T)2.0;
    if (kind == 1) { /* minmod */
        T v = theta < ONE ? theta : ONE;
        return v > ZERO ? v : ZERO;
    }
    if (kind == 2) { /* superbee */
        T a = TWO * theta;
        if (a > ONE) a = ONE;
        T b = theta < TWO ? theta : TWO;
        T v = a > b ? a : b;
        return v > ZERO ? v : ZERO;
    }
    if (kind == 3) { /* monotonized centered */
        T v = HALF * (ONE + theta);
        if (v > TWO) v = TWO;
        T tt = TWO * theta;
        if (tt < v) v = tt;
        return v > ZERO ? v : ZERO;
    }
    if (kind == 4) { /* van Leer */
        T a = CR_ABS(theta);
        return (theta + a) / (ONE + a);
    }
    return ONE;
}

/* Point-wise solvers.  W is (nw, m) row-major, s is (nw). */
static void CR_FN(solve)(int solver, const T *ql, const T *qr, int m, int normal,
                         const T *params, T *W, T *s)
{
    if (solver == CR_ADVECTION) { /* riemann.py:170-173 */
        W[0] = qr[0] - ql[0];
        s[0] = params[0];
        return;
    }
    if (solver == CR_ACOUSTICS) { /* riemann.py:116-133 */
        T c = params[0], Z = params[1], inv2z = params[2];
        T dp = qr[0] - ql[0];
        T dun = qr[normal] - ql[normal];
        T b1 = (Z * dun - dp) * inv2z;
        T b2 = (Z * dun + dp) * inv2z;
        for (int k = 0; k < m; ++k) { W[k] = (T)0; W[m + k] = (T)0; }
        W[0] = (-Z) * b1;
        W[normal] = b1;
        W[m + 0] = Z * b2;
        W[m + normal] = b2;
        s[0] = -c;
        s[1] = c;
        return;
    }
    if (solver == CR_SHALLOW_WATER) { /* riemann.py:136-167 */
        T g = params[0], half = params[1];
        int trans = 3 - normal;
        T hl = ql[0], hr = qr[0];
        T sl = CR_SQRT(hl);
        T sr = CR_SQRT(hr);
        T denom = sl + sr;
        T uhat = (ql[normal] / sl + qr[normal] / sr) / denom;
        T vhat = (ql[trans] / sl + qr[trans] / sr) / denom;
        T chat = CR_SQRT(g * (half * (hl + hr)));
        T dh = qr[0] - ql[0];
        T dhun = qr[normal] - ql[normal];
        T dhut = qr[trans] - ql[trans];
        T inv2c = half / chat;
        T a1 = ((uhat + chat) * dh - dhun) * inv2c;
        T a3 = (dhun - (uhat - chat) * dh) * inv2c;
        T a2 = dhut - vhat * dh;
        W[0] = a1;
        W[normal] = a1 * (uhat - chat);
        W[trans] = a1 * vhat;
        W[m + 0] = (T)0;
        W[m + normal] = (T)0;
        W[m + trans] = a2;
        W[2 * m + 0] = a3;
        W[2 * m + normal] = a3 * (uhat + chat);
        W[2 * m + trans] = a3 * vhat;
        s[0] = uhat - chat;
        s[1] = uhat;
        s[2] = uhat + chat;
        return;
    }
    /* CR_VC_ACOUSTICS: builder extension, heterogeneous medium carried as
     * two passive states (Z, c) at indices m-2, m-1. */
    {
        T Zl = ql[m - 2], Zr = qr[m - 2];
        T cl = ql[m - 1], cr = qr[m - 1];
        T dp = qr[0] - ql[0];
        T dun = qr[normal] - ql[normal];
        T denom = Zl + Zr;
        T a1 = (Zr * dun - dp) / denom;
        T a2 = (Zl * dun + dp) / denom;
        for (int k = 0; k < m; ++k) { W[k] = (T)0; W[m + k] = (T)0; }
        W[0] = (-Zl) * a1;
        W[normal] = a1;
        W[m + 0] = Zr * a2;
        W[m + normal] = a2;
        s[0] = -cl;
        s[1] = cr;
    }
}

/* sweep.py:183-263, one pencil list.  qin/qout are (m, padded_cells) flat,
 * sstride elements apart.  Returns the pencil-set max |s|. */
static T CR_FN(sweep_tile)(const T *qin, T *qout, int64_t sstride, int m,
                           const int64_t *bases, int64_t nbases, int64_t stride,
                           int64_t lo, int64_t hi, T dtdx, int normal,
                           const T *params, int limiter_id, int nw, int solver)
{
    const T ZERO = (T)0.0, HALF = (T)0.5, ONE = (T)1.0;
    T W[3][CR_MAXW * CR_MAXM], S[3][CR_MAXW];
    T am[3][CR_MAXM], ap[3][CR_MAXM];
    T ft_prev[CR_MAXM], ft_new[CR_MAXM], ql[CR_MAXM], qr[CR_MAXM];
    T smax = ZERO;
    for (int k = 0; k < CR_MAXM; ++k) ft_prev[k] = ZERO;
    for (int64_t b = 0; b < nbases; ++b) {
        int64_t base = bases[b];
        for (int64_t i = lo - 1; i < hi + 2; ++i) {
            int slot = (int)((i - (lo - 1)) % 3);
            int64_t off_l = base + (i - 1) * stride;
            int64_t off_r = base + i * stride;
            for (int k = 0; k < m; ++k) {
                ql[k] = qin[k * sstride + off_l];
                qr[k] = qin[k * sstride + off_r];
            }
            CR_FN(solve)(solver, ql, qr, m, normal, params, W[slot], S[slot]);
            for (int k = 0; k < m; ++k) { am[slot][k] = ZERO; ap[slot][k] = ZERO; }
            for (int p = 0; p < nw; ++p) {
                T sp = S[slot][p];
                T asp = CR_ABS(sp);
                if (asp > smax) smax = asp;
                if (sp < ZERO) {
                    for (int k = 0; k < m; ++k) am[slot][k] += sp * W[slot][p * m + k];
                } else if (sp > ZERO) {
                    for (int k = 0; k < m; ++k) ap[slot][k] += sp * W[slot][p * m + k];
                }
            }
            if (i >= lo + 1) {
                int s_mid = (int)((i - 1 - (lo - 1)) % 3);
                for (int k = 0; k < m; ++k) ft_new[k] = ZERO;
                for (int p = 0; p < nw; ++p) {
                    T sp = S[s_mid][p];
                    int s_up = sp > ZERO ? (int)((i - 2 - (lo - 1)) % 3) : slot;
                    T wn = ZERO, wu = ZERO;
                    for (int k = 0; k < m; ++k) {
                        T wk = W[s_mid][p * m + k];
                        wn += wk * wk;
                        wu += W[s_up][p * m + k] * wk;
                    }
                    T lim;
                    if (limiter_id == 0 || wn == ZERO)
                        lim = ONE;
                    else
                        lim = CR_FN(limiter_value)(wu / wn, limiter_id);
                    T asp = CR_ABS(sp);
                    T coef = ((HALF * asp) * (ONE - dtdx * asp)) * lim;
                    for (int k = 0; k < m; ++k) ft_new[k] += coef * W[s_mid][p * m + k];
                }
                if (i - 2 >= lo) {
                    int64_t c = base + (i - 2) * stride;
                    int s_left = (int)((i - 2 - (lo - 1)) % 3);
                    for (int k = 0; k < m; ++k) {
                        qout[k * sstride + c] = (qin[k * sstride + c]
                                                 - dtdx * (ap[s_left][k] + am[s_mid][k]))
                                                - dtdx * (ft_new[k] - ft_prev[k]);
                    }
                }
                for (int k = 0; k < m; ++k) ft_prev[k] = ft_new[k];
            }
        }
    }
    return smax;
}

#undef CR_FN
#undef CR_CAT
#undef CR_CAT2

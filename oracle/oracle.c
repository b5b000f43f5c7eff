/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arxiv 2203.09200 ("quarter sampling ... recursive FSR ... fast consistency
 * checks"): pixel-wise template-matching motion estimation (ME), the reverse
 * checks RME / RMC / FRMC, the nearest-neighbour check NNC and projection PR.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant with the CUDA library
 * (paper_2203_09200_b200/csrc, include/qs.h) and neither includes the other.
 *
 * Every function below follows the passage it cites.  Citations:
 *   PAPER.md:N  = line N of the paper text, with its section / equation.
 *   SPEC.md:N   = line N of the CPU specification written from the paper.
 *   Rk          = reading k of the register in DESIGN.md,
 *                 the binding interpretation where the paper is silent.
 *
 * No blocking, no fusion, no reordering: loops run in the order the
 * definitions are written (targets row-major, candidates in rank order,
 * template offsets row-major).
 *
 * Arithmetic:
 *   u8 reference  : integer terms, uint64 sums, exact cross-multiplied mean
 *                   comparison e1*n2 < e2*n1 (R1, R22).
 *   f32 reference : R23 -- c (u8) -> float exactly, d = fl(c - r), SAD term |d|,
 *                   SSD term fl(d*d) (built with -ffp-contract=off), fp32
 *                   accumulation in row-major offset order, mean fl(e/n),
 *                   fp32 '<' with ties by rank.  This is the kernel's precision
 *                   (task rule: a float that decides an integer -- the argmin --
 *                   is decided in the same precision on both sides).
 *   f64 mode      : the same definitions accumulated in fp64 (exact terms);
 *                   used only by the P15 error-bound pin.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

enum { OR_NOT_TARGET = 0, OR_INVALID = 1, OR_CANDIDATE = 2, OR_ACCEPTED = 3, OR_REJECTED = 4 };
enum { OR_REF_U8 = 0, OR_REF_F32 = 1, OR_REF_F32_ACC64 = 2 };

typedef struct {
    int32_t W, H;          /* frame width (cols) and height (rows) */
    int32_t Kh, Kw;        /* template size; offsets [-K/2, K-1-K/2] per axis (R2) */
    int32_t S;             /* search range, candidates [-S,S]^2 (R3) */
    int32_t min_support;   /* candidates with n < min_support are not admissible (R6) */
    int32_t ssd;           /* 0: SAD |d|, 1: SSD d^2 (R1) */
    int32_t ref_mode;      /* OR_REF_U8 | OR_REF_F32 | OR_REF_F32_ACC64 */
} or_params;

/* One matching error: integer sum (u8 refs), float sum (f32) or double (f64). */
typedef struct { uint64_t ei; float ef; double ed; int32_t n; } or_cost_t;

/* ------------------------------------------------------------------ */
/* Rank order of candidate vectors: (|a|+|b|, a, b) ascending (R7,     */
/* SPEC.md:246 "ties broken by (smaller |a|+|b|, then smaller a, then  */
/* smaller b)").                                                        */
/* ------------------------------------------------------------------ */
static int cmp_rank(const void *x, const void *y) {
    const int *p = (const int *)x, *q = (const int *)y;
    int l1 = abs(p[0]) + abs(p[1]), l2 = abs(q[0]) + abs(q[1]);
    if (l1 != l2) return l1 < l2 ? -1 : 1;
    if (p[0] != q[0]) return p[0] < q[0] ? -1 : 1;
    if (p[1] != q[1]) return p[1] < q[1] ? -1 : 1;
    return 0;
}

/* Writes the (2S+1)^2 candidates in rank order; returns the count. */
int or_rank_list(int32_t S, int32_t *alpha, int32_t *beta) {
    int n = (2 * S + 1) * (2 * S + 1);
    int *v = (int *)malloc(sizeof(int) * 2 * (size_t)n);
    if (!v) return -1;
    int k = 0;
    for (int a = -S; a <= S; ++a)
        for (int b = -S; b <= S; ++b) { v[2 * k] = a; v[2 * k + 1] = b; ++k; }
    qsort(v, (size_t)n, sizeof(int) * 2, cmp_rank);
    for (int i = 0; i < n; ++i) { alpha[i] = v[2 * i]; beta[i] = v[2 * i + 1]; }
    free(v);
    return n;
}

static int in_frame(const or_params *P, int y, int x) {
    return y >= 0 && y < P->H && x >= 0 && x < P->W;
}

static float ref_f(const void *ref, const or_params *P, int y, int x) {
    return ((const float *)ref)[(size_t)y * P->W + x];
}
static int ref_u(const void *ref, const or_params *P, int y, int x) {
    return ((const uint8_t *)ref)[(size_t)y * P->W + x];
}

/* Add one term phi(a - b) where a is the u8 current sample and b the reference
 * sample (forward) -- or a is the reference and b the current sample (reverse);
 * phi is symmetric and fl(a-b) = -fl(b-a), so both orders give the same term. */
static void add_term(const or_params *P, or_cost_t *c, int cur_v, const void *ref, int ry, int rx) {
    if (P->ref_mode == OR_REF_U8) {
        int64_t d = (int64_t)cur_v - (int64_t)ref_u(ref, P, ry, rx);
        c->ei += (uint64_t)(P->ssd ? d * d : (d < 0 ? -d : d));
    } else if (P->ref_mode == OR_REF_F32) {
        float d = (float)cur_v - ref_f(ref, P, ry, rx);   /* d = fl(c - r) */
        float t = P->ssd ? d * d : fabsf(d);              /* fl(d*d), no FMA contraction */
        c->ef = c->ef + t;                                /* row-major fp32 accumulation */
    } else {
        double d = (double)cur_v - (double)ref_f(ref, P, ry, rx);
        double t = P->ssd ? d * d : fabs(d);
        c->ed = c->ed + t;
    }
    c->n += 1;
}

/* Forward matching error of target p=(py,px) for v=(a,b) (§2.2
 * "pixel-wise template matching using the already reconstructed past frames
 * and the measured data from the current frame"):
 *   e(p,v) = sum_{q in T_p(v)} phi(cur(q) - ref(q+v)),  n = |T_p(v)|,
 *   T_p(v) = { q = p+o : q in frame, cur_mask(q)=1, q+v in frame }   (R5, R6),
 * o running row-major over [-Kh/2, Kh-1-Kh/2] x [-Kw/2, Kw-1-Kw/2]    (R2). */
or_cost_t or_cost_fwd(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                      int py, int px, int a, int b) {
    or_cost_t c; memset(&c, 0, sizeof c);
    int oy0 = -(P->Kh / 2), oy1 = P->Kh - 1 - P->Kh / 2;
    int ox0 = -(P->Kw / 2), ox1 = P->Kw - 1 - P->Kw / 2;
    for (int oy = oy0; oy <= oy1; ++oy)
        for (int ox = ox0; ox <= ox1; ++ox) {
            int qy = py + oy, qx = px + ox;
            if (!in_frame(P, qy, qx)) continue;
            if (!mask[(size_t)qy * P->W + qx]) continue;
            if (!in_frame(P, qy + a, qx + b)) continue;
            add_term(P, &c, cur[(size_t)qy * P->W + qx], ref, qy + a, qx + b);
        }
    return c;
}

/* Reverse matching error at x=(xy,xx) for reverse vector u=(a,b) (PAPER.md:71
 * §2.2 "motion vectors in the reverse direction"; R9):
 * the dense reference template at x against the sparse current frame at x+u:
 *   e'(x,u) = sum_{q} phi(ref(q) - cur(q+u)) over q = x+o with q in frame,
 *   q+u in frame and cur_mask(q+u) = 1, o row-major.  x itself may lie
 * outside the frame.  The caller treats n' < min_support as the SENTINEL. */
or_cost_t or_cost_rev(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                      int xy, int xx, int a, int b) {
    or_cost_t c; memset(&c, 0, sizeof c);
    int oy0 = -(P->Kh / 2), oy1 = P->Kh - 1 - P->Kh / 2;
    int ox0 = -(P->Kw / 2), ox1 = P->Kw - 1 - P->Kw / 2;
    for (int oy = oy0; oy <= oy1; ++oy)
        for (int ox = ox0; ox <= ox1; ++ox) {
            int qy = xy + oy, qx = xx + ox;
            if (!in_frame(P, qy, qx)) continue;
            int sy = qy + a, sx = qx + b;
            if (!in_frame(P, sy, sx)) continue;
            if (!mask[(size_t)sy * P->W + sx]) continue;
            add_term(P, &c, cur[(size_t)sy * P->W + sx], ref, qy, qx);
        }
    return c;
}

/* Mean comparison "c1 has a strictly smaller mean than c2" (R1):
 * u8: exact e1*n2 < e2*n1; f32: fl(e1/n1) < fl(e2/n2) (R23); f64: e1/n1 < e2/n2. */
static int mean_less(const or_params *P, const or_cost_t *c1, const or_cost_t *c2) {
    if (P->ref_mode == OR_REF_U8)
        return c1->ei * (uint64_t)c2->n < c2->ei * (uint64_t)c1->n;
    if (P->ref_mode == OR_REF_F32) {
        float m1 = c1->ef / (float)c1->n;
        float m2 = c2->ef / (float)c2->n;
        return m1 < m2;
    }
    return c1->ed / (double)c1->n < c2->ed / (double)c2->n;
}

static int cost_equal(const or_params *P, const or_cost_t *c1, const or_cost_t *c2) {
    if (c1->n != c2->n) return 0;
    if (P->ref_mode == OR_REF_U8) return c1->ei == c2->ei;
    if (P->ref_mode == OR_REF_F32) return c1->ef == c2->ef;
    return c1->ed == c2->ed;
}

static void store_err(const or_params *P, void *err, size_t i, const or_cost_t *c) {
    if (P->ref_mode == OR_REF_U8) ((uint32_t *)err)[i] = (uint32_t)c->ei;
    else if (P->ref_mode == OR_REF_F32) ((float *)err)[i] = c->ef;
    else ((double *)err)[i] = c->ed;
}

static or_cost_t load_err(const or_params *P, const void *err, const uint8_t *count, size_t i) {
    or_cost_t c; memset(&c, 0, sizeof c);
    if (P->ref_mode == OR_REF_U8) c.ei = ((const uint32_t *)err)[i];
    else if (P->ref_mode == OR_REF_F32) c.ef = ((const float *)err)[i];
    else c.ed = ((const double *)err)[i];
    c.n = count[i];
    return c;
}

static int check_params(const or_params *P) {
    if (P->W <= 0 || P->H <= 0 || P->Kh <= 0 || P->Kw <= 0 || P->S < 0 || P->S > 127) return -1;
    if (P->min_support < 1) return -1;
    if (P->ref_mode < 0 || P->ref_mode > 2) return -1;
    return 0;
}

/* ------------------------------------------------------------------ */
/* ME (§2.2; R4-R7).                       */
/* For every target p (cur_mask(p) = 0, "For any missing pixel", R4) in */
/* rows [y_begin, y_end): scan v in rank order, skip v with n <         */
/* min_support (R6), keep v if it has a strictly smaller mean than the  */
/* best so far (strict '<' in rank order = the tie-break of R7).        */
/* Outputs: alpha (rows), beta (cols) (R8), err, count, status.         */
/* Non-targets get status NOT_TARGET and zeros; targets with no         */
/* admissible candidate get INVALID and zeros.                          */
/* ------------------------------------------------------------------ */
int or_me_search(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                 int32_t y_begin, int32_t y_end,
                 int8_t *alpha, int8_t *beta, void *err, uint8_t *count, uint8_t *status) {
    if (check_params(P)) return -1;
    int nc = (2 * P->S + 1) * (2 * P->S + 1);
    int32_t *ra = (int32_t *)malloc(sizeof(int32_t) * (size_t)nc);
    int32_t *rb = (int32_t *)malloc(sizeof(int32_t) * (size_t)nc);
    if (!ra || !rb) { free(ra); free(rb); return -2; }
    or_rank_list(P->S, ra, rb);
    if (y_begin < 0) y_begin = 0;
    if (y_end > P->H) y_end = P->H;
    for (int py = y_begin; py < y_end; ++py)
        for (int px = 0; px < P->W; ++px) {
            size_t i = (size_t)py * P->W + px;
            or_cost_t zero; memset(&zero, 0, sizeof zero);
            alpha[i] = 0; beta[i] = 0; count[i] = 0; store_err(P, err, i, &zero);
            if (mask[i]) { status[i] = OR_NOT_TARGET; continue; }
            int have = 0, ba = 0, bb = 0;
            or_cost_t best; memset(&best, 0, sizeof best);
            for (int k = 0; k < nc; ++k) {
                or_cost_t c = or_cost_fwd(P, cur, mask, ref, py, px, ra[k], rb[k]);
                if (c.n < P->min_support) continue;
                if (!have || mean_less(P, &c, &best)) { best = c; ba = ra[k]; bb = rb[k]; have = 1; }
            }
            if (!have) { status[i] = OR_INVALID; continue; }
            alpha[i] = (int8_t)ba; beta[i] = (int8_t)bb; count[i] = (uint8_t)best.n;
            store_err(P, err, i, &best);
            status[i] = OR_CANDIDATE;
        }
    free(ra); free(rb);
    return 0;
}

/* Entries a check may examine: "Each check reads only entries whose status is
 * CANDIDATE or ACCEPTED" (checks compose by narrowing; R16). */
static int checkable(uint8_t s) { return s == OR_CANDIDATE || s == OR_ACCEPTED; }

/* ------------------------------------------------------------------ */
/* RMC / FRMC (§3.1.1; R11, R12, R17) */
/* At x = p+v the reverse costs for u = -v + delta are evaluated; the   */
/* entry is REJECTED iff some delta != 0 with an admissible cost has a  */
/* strictly smaller mean than delta = 0 ("If any of the red arrows has  */
/* the lowest cost ... rejected"), else ACCEPTED.  delta ranges over    */
/* offs x offs (FRMC: {-7,-3,-1,0,1,3,7}) or [-S,S]^2     */
/* (RMC).  The delta = 0 cost is rc(p+v, -v), which equals the forward  */
/* (e, n) exactly (identity P4); the oracle recomputes it, uses the     */
/* recomputed value, and (verify_p4 != 0) returns -5 if it differs from */
/* the stored forward cost.  *evals += |delta set| per checked entry.   */
/* ------------------------------------------------------------------ */
static int reverse_check_grid(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                              const int32_t *offs, int32_t n_offs, int32_t y_begin, int32_t y_end,
                              const int8_t *alpha, const int8_t *beta, const void *err, const uint8_t *count,
                              uint8_t *status, uint64_t *evals, int verify_p4) {
    if (y_begin < 0) y_begin = 0;
    if (y_end > P->H) y_end = P->H;
    for (int py = y_begin; py < y_end; ++py)
        for (int px = 0; px < P->W; ++px) {
            size_t i = (size_t)py * P->W + px;
            if (!checkable(status[i])) continue;
            int a = alpha[i], b = beta[i];
            int xy = py + a, xx = px + b;
            or_cost_t c0 = or_cost_rev(P, cur, mask, ref, xy, xx, -a, -b);
            if (verify_p4) {
                or_cost_t fw = load_err(P, err, count, i);
                if (!cost_equal(P, &c0, &fw)) return -5;   /* P4 violated: inputs inconsistent */
            }
            int reject = 0;
            for (int j = 0; j < n_offs; ++j)
                for (int k = 0; k < n_offs; ++k) {
                    int dy = offs[j], dx = offs[k];
                    if (dy == 0 && dx == 0) continue;
                    or_cost_t c = or_cost_rev(P, cur, mask, ref, xy, xx, -a + dy, -b + dx);
                    if (c.n < P->min_support) continue;       /* SENTINEL never rejects (R11) */
                    if (mean_less(P, &c, &c0)) reject = 1;
                }
            if (evals) *evals += (uint64_t)n_offs * (uint64_t)n_offs;
            status[i] = reject ? OR_REJECTED : OR_ACCEPTED;
        }
    return 0;
}

int or_frmc(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
            const int32_t *offsets, int32_t n_offsets, int32_t y_begin, int32_t y_end,
            const int8_t *alpha, const int8_t *beta, const void *err, const uint8_t *count,
            uint8_t *status, uint64_t *evals, int32_t verify_p4) {
    if (check_params(P)) return -1;
    int has0 = 0;
    for (int j = 0; j < n_offsets; ++j) {
        if (offsets[j] == 0) has0 = 1;
        if (offsets[j] < -P->S || offsets[j] > P->S) return -1;
    }
    if (!has0 || n_offsets <= 0) return -1;
    return reverse_check_grid(P, cur, mask, ref, offsets, n_offsets, y_begin, y_end,
                              alpha, beta, err, count, status, evals, verify_p4);
}

int or_rmc(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
           int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
           const void *err, const uint8_t *count, uint8_t *status, uint64_t *evals, int32_t verify_p4) {
    if (check_params(P)) return -1;
    int n = 2 * P->S + 1;
    int32_t *offs = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!offs) return -2;
    for (int j = 0; j < n; ++j) offs[j] = j - P->S;
    int r = reverse_check_grid(P, cur, mask, ref, offs, n, y_begin, y_end,
                               alpha, beta, err, count, status, evals, verify_p4);
    free(offs);
    return r;
}

/* RME (§2.2 "the motion vectors in the reverse direction are
 * calculated using an additional reverse motion estimation ... Only when both
 * motion vectors coincide, the motion vector is accepted"; SPEC.md:297-305;
 * R10): at x = p+v, the reverse argmin over u in [-S,S]^2, scanned in rank
 * order with strict '<' and SENTINELs skipped; ACCEPTED iff argmin == -v. */
int or_rme(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
           int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
           const void *err, const uint8_t *count, uint8_t *status, uint64_t *evals) {
    if (check_params(P)) return -1;
    int nc = (2 * P->S + 1) * (2 * P->S + 1);
    int32_t *ra = (int32_t *)malloc(sizeof(int32_t) * (size_t)nc);
    int32_t *rb = (int32_t *)malloc(sizeof(int32_t) * (size_t)nc);
    if (!ra || !rb) { free(ra); free(rb); return -2; }
    or_rank_list(P->S, ra, rb);
    (void)err; (void)count;
    if (y_begin < 0) y_begin = 0;
    if (y_end > P->H) y_end = P->H;
    for (int py = y_begin; py < y_end; ++py)
        for (int px = 0; px < P->W; ++px) {
            size_t i = (size_t)py * P->W + px;
            if (!checkable(status[i])) continue;
            int a = alpha[i], b = beta[i];
            int xy = py + a, xx = px + b;
            int have = 0, ua = 0, ub = 0;
            or_cost_t best; memset(&best, 0, sizeof best);
            for (int k = 0; k < nc; ++k) {
                or_cost_t c = or_cost_rev(P, cur, mask, ref, xy, xx, ra[k], rb[k]);
                if (c.n < P->min_support) continue;
                if (!have || mean_less(P, &c, &best)) { best = c; ua = ra[k]; ub = rb[k]; have = 1; }
            }
            if (evals) *evals += (uint64_t)nc;
            status[i] = (have && ua == -a && ub == -b) ? OR_ACCEPTED : OR_REJECTED;
        }
    free(ra); free(rb);
    return 0;
}

/* ------------------------------------------------------------------ */
/* NNC (§3.1.2, Eq. (1) at PAPER.md:110-113;          */
/* SPEC.md:324-341; R14, R15).                                          */
/* (1) Filter, Eq. (1): for every valid entry p (status >= CANDIDATE,   */
/*     whatever its accept state), each component's median over the     */
/*     valid entries of the in-frame 3x3 window centred on p (centre    */
/*     included), lower median for even counts.                         */
/* (2) Decide: an entry with status CANDIDATE or ACCEPTED is REJECTED   */
/*     iff some in-frame valid 4-neighbour nb has                       */
/*     |a~(p)-a~(nb)| + |b~(p)-b~(nb)| > threshold (paper: "at most     */
/*     one"), else ACCEPTED.  Rows [y_begin, y_end) are decided; the    */
/*     filter reads the whole frame.                                    */
/* ------------------------------------------------------------------ */
static int cmp_int(const void *x, const void *y) {
    int a = *(const int *)x, b = *(const int *)y;
    return (a > b) - (a < b);
}

/* mode 0: the reading above (R15).  mode 1: the other reading of "at most one for each neighboring */
/* pair" (SPEC.md:369 open question; R30): the filtered vectors of the in-    */
/* frame valid 4-neighbours are compared with EACH OTHER (every unordered pair of them, the centre    */
/* not compared); REJECTED iff some pair differs by more than threshold, else ACCEPTED.               */
int or_nnc_mode(int32_t W, int32_t H, int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
                uint8_t *status, int32_t threshold, int32_t mode) {
    if (W <= 0 || H <= 0 || threshold < 0 || mode < 0 || mode > 1) return -1;
    size_t N = (size_t)W * H;
    int *fa = (int *)malloc(sizeof(int) * N), *fb = (int *)malloc(sizeof(int) * N);
    uint8_t *valid = (uint8_t *)malloc(N);
    if (!fa || !fb || !valid) { free(fa); free(fb); free(valid); return -2; }
    for (size_t i = 0; i < N; ++i) valid[i] = status[i] >= OR_CANDIDATE;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t i = (size_t)y * W + x;
            fa[i] = fb[i] = 0;
            if (!valid[i]) continue;
            int la[9], lb[9], n = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int yy = y + dy, xx = x + dx;
                    if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                    size_t j = (size_t)yy * W + xx;
                    if (!valid[j]) continue;
                    la[n] = alpha[j]; lb[n] = beta[j]; ++n;
                }
            qsort(la, (size_t)n, sizeof(int), cmp_int);
            qsort(lb, (size_t)n, sizeof(int), cmp_int);
            fa[i] = la[(n - 1) / 2];
            fb[i] = lb[(n - 1) / 2];
        }
    if (y_begin < 0) y_begin = 0;
    if (y_end > H) y_end = H;
    static const int NB[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};
    for (int y = y_begin; y < y_end; ++y)
        for (int x = 0; x < W; ++x) {
            size_t i = (size_t)y * W + x;
            if (!checkable(status[i])) continue;
            int reject = 0;
            size_t nbj[4];
            int nn = 0;
            for (int k = 0; k < 4; ++k) {
                int yy = y + NB[k][0], xx = x + NB[k][1];
                if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                size_t j = (size_t)yy * W + xx;
                if (!valid[j]) continue;
                nbj[nn++] = j;
            }
            if (mode == 0) {
                for (int k = 0; k < nn; ++k) {
                    size_t j = nbj[k];
                    if (abs(fa[i] - fa[j]) + abs(fb[i] - fb[j]) > threshold) reject = 1;
                }
            } else {
                for (int k = 0; k < nn; ++k)
                    for (int l = k + 1; l < nn; ++l) {
                        size_t j = nbj[k], m = nbj[l];
                        if (abs(fa[j] - fa[m]) + abs(fb[j] - fb[m]) > threshold) reject = 1;
                    }
            }
            status[i] = reject ? OR_REJECTED : OR_ACCEPTED;
        }
    free(fa); free(fb); free(valid);
    return 0;
}

int or_nnc(int32_t W, int32_t H, int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
           uint8_t *status, int32_t threshold) {
    return or_nnc_mode(W, H, y_begin, y_end, alpha, beta, status, threshold, 0);
}

/* Filtered field of Eq. (1) alone (for pins); undefined entries get 0 and def=0. */
int or_median_field(int32_t W, int32_t H, const int8_t *alpha, const int8_t *beta, const uint8_t *status,
                    int32_t *fa, int32_t *fb, uint8_t *def) {
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t i = (size_t)y * W + x;
            fa[i] = fb[i] = 0; def[i] = 0;
            if (status[i] < OR_CANDIDATE) continue;
            int la[9], lb[9], n = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int yy = y + dy, xx = x + dx;
                    if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                    size_t j = (size_t)yy * W + xx;
                    if (status[j] < OR_CANDIDATE) continue;
                    la[n] = alpha[j]; lb[n] = beta[j]; ++n;
                }
            qsort(la, (size_t)n, sizeof(int), cmp_int);
            qsort(lb, (size_t)n, sizeof(int), cmp_int);
            fa[i] = la[(n - 1) / 2]; fb[i] = lb[(n - 1) / 2]; def[i] = 1;
        }
    return 0;
}

/* ------------------------------------------------------------------ */
/* PR (§2.2 "values for some of the missing pixels ... can  */
/* be found by following their motion vector into the past. If a       */
/* measurement is available at the corresponding position in the past  */
/* frame, it is projected ... In case projections from more than one    */
/* past frame are available, these are averaged.";     */
/* R18): for each ACCEPTED p, q = p+v; if q in frame and                */
/* past_mask(q) = 1: sum(p) += past_val(q), cnt(p) += 1.  Accumulates   */
/* into caller-zeroed buffers; the average sum/cnt is the consumer's.   */
/* ------------------------------------------------------------------ */
int or_project(int32_t W, int32_t H, int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
               const uint8_t *status, const uint8_t *past_val, const uint8_t *past_mask,
               uint32_t *sum, uint8_t *cnt) {
    if (W <= 0 || H <= 0) return -1;
    if (y_begin < 0) y_begin = 0;
    if (y_end > H) y_end = H;
    for (int y = y_begin; y < y_end; ++y)
        for (int x = 0; x < W; ++x) {
            size_t i = (size_t)y * W + x;
            if (status[i] != OR_ACCEPTED) continue;
            int qy = y + alpha[i], qx = x + beta[i];
            if (qy < 0 || qy >= H || qx < 0 || qx >= W) continue;
            size_t j = (size_t)qy * W + qx;
            if (!past_mask[j]) continue;
            sum[i] += past_val[j];
            cnt[i] += 1;
        }
    return 0;
}

/* Single-cost probes for pins and near-tie classification in tests. */
int or_probe_fwd(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                 int32_t py, int32_t px, int32_t a, int32_t b, uint64_t *ei, float *ef, double *ed) {
    or_cost_t c = or_cost_fwd(P, cur, mask, ref, py, px, a, b);
    *ei = c.ei; *ef = c.ef; *ed = c.ed;
    return c.n;
}

int or_probe_rev(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                 int32_t xy, int32_t xx, int32_t a, int32_t b, uint64_t *ei, float *ef, double *ed) {
    or_cost_t c = or_cost_rev(P, cur, mask, ref, xy, xx, a, b);
    *ei = c.ei; *ef = c.ef; *ed = c.ed;
    return c.n;
}

/*
 * qs.h -- C ABI of libqs: the B200 (sm_100a) hot path of arxiv 2203.09200,
 * "recursive FSR for quarter-sampled video with fast consistency checks".
 *
 * The path, per (current frame t, reference distance d) pair (PAPER.md:30-41
 * Fig. 1, :68-74 §2.2, :99-115 §3.1):
 *   ME  (qs_me_search)     pixel-wise template matching of the current frame's
 *                          measured pixels against the previous reconstruction
 *   CC  (qs_nnc, qs_frmc,  consistency checks that reject untrustworthy vectors
 *        qs_reverse_check) (NNC, FRMC = the paper's; RME, RMC = the literature's)
 *   PR  (qs_project)       projection of past measurements along accepted vectors
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - Pointers to image / field data are DEVICE pointers owned by the caller.
 *   The library allocates nothing per call and keeps no pointer after return;
 *   work is ENQUEUED on `stream` (a cudaStream_t passed as void*, NULL = legacy
 *   default stream).  The caller keeps buffers alive until the stream reaches
 *   the work.  The only allocations are one-time per-device candidate tables
 *   (rank LUTs, <= 4225 entries per S) built on first use.
 * - Images are row-major [rows][cols].  Frame coordinates p = (m, n) = (row, col)
 *   ("(alpha_mn, beta_mn)"); a motion vector v = (alpha, beta) =
 *   (rows, cols) points from the current pixel p to p+v in the past frame
 *   (Fig. 2(a) "motion vector field from frame f(t) to f(t-1)").
 * - Row windows (qs_roi): every buffer passed to one call holds the global
 *   frame rows [buf_y0, buf_y0 + buf_rows); row r of a buffer is global row
 *   buf_y0 + r.  Work is produced for global rows [y_begin, y_end).  All border
 *   rules use the FULL frame (frame_w, frame_h) -- a band edge is not a border
 *   (reading R25).  roi is required (it carries the frame size); QS_EINVAL if NULL.
 * - Pitches: image pitches are in BYTES and must be multiples of 16, base
 *   pointers 16-byte aligned (QS_EALIGN otherwise); the qs_field pitch is in
 *   ELEMENTS and shared by its five planes.
 * - Errors: arguments are validated synchronously before anything is enqueued;
 *   on failure nothing is written and a negative code is returned, with a
 *   message available from qs_last_error() (thread-local).  A failed launch
 *   returns QS_ECUDA; faults inside a kernel surface at the caller's next
 *   synchronisation of `stream`.  No C++ exception crosses the ABI; nothing
 *   calls exit() or abort().
 * - Determinism: results are bit-identical for any stream, launch order or row
 *   banding.  Results are a pure function of the inputs.
 * - Concurrency: all entry points are re-entrant; calls on different streams
 *   may overlap.
 */
#ifndef QS_H_
#define QS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes. */
enum {
    QS_OK = 0,
    QS_EINVAL = -1,   /* bad parameter: K, S, min_support, offsets, mode, NULL pointer */
    QS_EDIM = -2,     /* bad frame size (non-positive or odd), roi outside the frame,
                         buffer window missing required halo rows, workspace too small */
    QS_EALIGN = -3,   /* base pointer or pitch not 16-byte aligned */
    QS_ECUDA = -4     /* a CUDA launch / runtime call failed */
};

/* Field status (R4, R6, R16). */
enum {
    QS_NOT_TARGET = 0,   /* measured pixel in the current frame: no vector (R4) */
    QS_INVALID = 1,      /* target with no admissible candidate (n < min_support for all v; R6) */
    QS_CANDIDATE = 2,    /* ME result, not yet checked */
    QS_ACCEPTED = 3,     /* passed the last check run on it */
    QS_REJECTED = 4      /* failed a check (never reconsidered) */
};

enum { QS_SAD = 0, QS_SSD = 1 };          /* matching error phi (R1) */
enum { QS_REF_U8 = 0, QS_REF_F32 = 1 };   /* element type of the reference frame (R20) */
enum { QS_RME = 0, QS_RMC = 1 };          /* literature / intermediate reverse checks */

/* ME parameters.
 *   K_h, K_w     template size; offsets o in [-K/2, K-1-K/2] per axis (R2).  This
 *                build supports square templates 1 <= K_h == K_w <= 9 (QS_EINVAL else).
 *   S            search range: candidates v in [-S, S]^2 (PAPER.md:104 uses S=9;
 *                R3).  0 <= S <= 32.
 *   min_support  candidates whose support n = |T_p(v)| < min_support are not
 *                admissible (R6); >= 1.
 *   err          QS_SAD or QS_SSD (R1).
 *   ref_type     QS_REF_U8 (uint8 reference) or QS_REF_F32 (float32 reference). */
typedef struct {
    int32_t K_h, K_w;
    int32_t S;
    int32_t min_support;
    int32_t err;
    int32_t ref_type;
} qs_me_params;

typedef struct {
    int32_t frame_w, frame_h;   /* full frame: every border rule uses these (R25); even, > 0 */
    int32_t y_begin, y_end;     /* global rows to produce, 0 <= y_begin <= y_end <= frame_h */
    int32_t buf_y0, buf_rows;   /* global row of buffer row 0; number of rows held */
} qs_roi;

/* Motion field, structure of arrays [rows][pitch].
 *   alpha, beta  int8 vector (rows, cols); meaningful iff status >= QS_CANDIDATE
 *   err          matching error e of the chosen vector: uint32 (u8 reference) or
 *                float (f32 reference); e = sum of phi over the support
 *   count        support n = |T_p(v)| (uint8)
 *   status       QS_NOT_TARGET .. QS_REJECTED (uint8)
 * Non-targets and INVALID entries hold alpha = beta = err = count = 0. */
typedef struct {
    int8_t *alpha;
    int8_t *beta;
    void *err;
    uint8_t *count;
    uint8_t *status;
    int64_t pitch;   /* in elements, shared by the five planes */
} qs_field;

/* NNC readings of PAPER.md:114 "at most one for each neighboring pair" (R15 / R30). */
#define QS_NNC_CENTRE 1   /* the filtered centre against each filtered 4-neighbour (headline, R15) */
#define QS_NNC_PAIRS 2    /* the filtered 4-neighbours against each other (R30) */

/* Checks fused into qs_me_search (NULL = ME only).
 *   nnc            0 = no NNC; QS_NNC_CENTRE / QS_NNC_PAIRS = run NNC
 *                  after ME with that reading; other values QS_EINVAL
 *   nnc_threshold  accept iff |da~| + |db~| <= threshold for every tested
 *                  neighbour (paper: "at most one" -> 1)
 *   frmc           run FRMC on the entries left checkable
 *   offsets        HOST array of per-axis FRMC offsets; must contain 0 and
 *                  satisfy |o| <= S (paper: {-7,-3,-1,0,1,3,7})
 *   n_offsets      1..15
 * With nnc and frmc both set this is the paper's cascade NNC -> FRMC: NNC
 * rejects, FRMC decides the NNC survivors (R16). */
typedef struct {
    int32_t nnc, nnc_threshold;
    int32_t frmc;
    const int8_t *offsets;
    int32_t n_offsets;
} qs_checks;

/* ---------------------------------------------------------------------------
 * Workspace.  qs_me_search and qs_reverse_check(QS_RME) need a caller-owned
 * device scratch buffer of at least the returned size (16-byte aligned).
 * Returns QS_OK and writes *bytes, or an error code for invalid arguments.
 * ------------------------------------------------------------------------- */
int qs_workspace_size(const qs_roi *roi, int32_t frame_w, int32_t frame_h, const qs_me_params *p,
                      size_t *bytes);

/* ---------------------------------------------------------------------------
 * qs_me_search -- motion estimation by exhaustive template matching
 * (§2.2: "the motion estimation is performed by a pixel-wise
 * template matching using the already reconstructed past frames and the
 * measured data from the current frame").
 *
 * For every target p (cur_mask(p) == 0, "for any missing pixel", R4) in rows
 * [y_begin, y_end) and every v in [-S,S]^2:
 *     e(p,v) = sum_{q in T_p(v)} phi(cur(q) - ref(q+v)),  n(p,v) = |T_p(v)|,
 *     T_p(v) = { q = p+o : q in frame, cur_mask(q) = 1, q+v in frame }.
 * The chosen v minimises the mean e/n over admissible candidates (n >=
 * min_support), ties broken by (|alpha|+|beta|, alpha, beta) ascending (R7).
 * Mean comparison: exact for uint8 references (integer cross-multiplication).
 * For float32 references the result is the definition's in fp32 arithmetic
 * (R23): terms fl(c - r), |d| or fl(d*d), summed in row-major template order,
 * compared by fl(e/n), ties by rank -- bit-identical to a sequential
 * implementation.  The search sums in a faster blocked order and certifies
 * each winner against an error bound; outputs it cannot certify are
 * recomputed in the definition's order (
 * qs_certify_stats counts them).  err is the row-major fp32 sum.
 *
 *   cur, cur_mask  uint8 [rows][cur_pitch]: current sampled frame (values read
 *                  only where cur_mask == 1) and its quarter mask in {0,1}
 *   ref            uint8 or float32 [rows][ref_pitch]: previous reconstruction
 *   roi            row window (required: it carries the frame size); buffers must hold rows
 *                  [y_begin - K/2 - S - 2, y_end + K + S + 2) clipped to the frame
 *                  (the +2 covers the NNC halo when `fuse` is set)
 *   fuse           NULL = ME only (statuses NOT_TARGET / INVALID / CANDIDATE);
 *                  otherwise the checks of qs_checks run on rows [y_begin, y_end).
 *                  NNC needs vectors 2 rows beyond the roi: ME then also runs on
 *                  rows [y_begin-2, y_end+2) (clipped to the frame), which the
 *                  field buffers must hold, but only rows [y_begin, y_end) of
 *                  `out` are written (the halo vectors stay in the workspace),
 *                  so adjacent rois may share one field buffer and run on
 *                  different streams.
 *   out            field planes (buffer window of the roi)
 *   eval_count     nullable device counter; FRMC adds |offsets|^2 per checked
 *                  entry (definitional count, R17)
 *   workspace      device scratch of qs_workspace_size() bytes
 * ------------------------------------------------------------------------- */
int qs_me_search(const uint8_t *cur, const uint8_t *cur_mask, int64_t cur_pitch,
                 const void *ref, int64_t ref_pitch, const qs_roi *roi,
                 const qs_me_params *p, const qs_checks *fuse, qs_field *out,
                 unsigned long long *eval_count, void *workspace, size_t workspace_bytes,
                 void *stream);

/* ---------------------------------------------------------------------------
 * qs_me_search_refs -- qs_me_search for the pairs (cur, refs[i]) of one frame,
 * i = 0..n_refs-1 (the d = 1..3 references of PAPER.md:131 "the last three
 * frames"): the same results as n_refs calls
 * of qs_me_search(cur, cur_mask, cur_pitch, refs[i], ref_pitch, roi, p, fuse,
 * &outs[i], ...), with ME and the fused checks of all references in ONE launch
 * per kernel (K = 8 with the paper's FRMC offsets or no FRMC; other settings run
 * the calls one by one).  The CTAs of the references for one tile and chunk run
 * side by side (the current frame's tile is read from L2 by all of them; no
 * per-reference tail between launches).
 *
 *   refs        HOST array of n_refs DEVICE reference planes (same type, pitch)
 *   outs        HOST array of n_refs fields (each with its own planes / pitch), or NULL
 *               with a projection: "projection-only" -- the fields are not written, only
 *               sum / cnt (the vectors never leave the chip except
 *               as the projection overlay); needs K = 8 and no or the paper's FRMC offsets
 *               (QS_EINVAL otherwise)
 *   proj        NULL, or the projection PR fused into the same launch: reference i's
 *               ACCEPTED entries project past_val[i] / past_mask[i] into sum / cnt
 *               exactly as qs_project(&outs[i], past_val[i], past_mask[i], ...) for
 *               i = 0..n_refs-1 would (integer sums: the result does not depend on
 *               the order); the past planes hold the rows qs_project needs.  cnt must be
 *               4-byte aligned with acc_pitch % 4 == 0, and
 *               every cnt byte must stay < 256 (it does for <= 255 references on a
 *               zeroed plane).
 *   eval_count  nullable device counter: the sum over the references
 *   workspace   n_refs slots of qs_workspace_size() bytes each
 * n_refs = 0 is a no-op; any n_refs >= 1 is accepted (launched in groups of 4).
 * Errors as qs_me_search; a failing group leaves later references untouched.
 * ------------------------------------------------------------------------- */
typedef struct {
    const uint8_t *const *past_val;    /* HOST array of n_refs DEVICE planes: frame t-d measurements */
    const uint8_t *const *past_mask;   /* HOST array of n_refs DEVICE planes: their masks */
    int64_t past_pitch;                /* bytes, shared by every past plane */
    uint32_t *sum;                     /* [rows][acc_pitch], accumulated (caller-zeroed per frame) */
    uint8_t *cnt;                      /* [rows][acc_pitch], accumulated */
    int64_t acc_pitch;                 /* elements */
} qs_projection;

int qs_me_search_refs(const uint8_t *cur, const uint8_t *cur_mask, int64_t cur_pitch, int32_t n_refs,
                      const void *const *refs, int64_t ref_pitch, const qs_roi *roi, const qs_me_params *p,
                      const qs_checks *fuse, qs_field *outs, const qs_projection *proj,
                      unsigned long long *eval_count, void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * qs_reverse_check -- the literature's RME (mode QS_RME; PAPER.md:71-72:
 * "the motion vectors in the reverse direction are calculated using an
 * additional reverse motion estimation (RME). Only when both motion vectors
 * coincide, the motion vector is accepted.") and the intermediate RMC (mode
 * QS_RMC; "testing the same number of motions vectors as in RME
 * but placing them symmetrically around the motion vector pointing back").
 *
 * Reverse cost at x = p+v for reverse vector u (R9):
 *     e'(x,u) = sum phi(ref(q) - cur(q+u)) over q = x+o with q in frame,
 *               q+u in frame, cur_mask(q+u) = 1;  SENTINEL if n' < min_support.
 * RME: ACCEPTED iff the reverse argmin over u in [-S,S]^2 (rank order, strict
 *      '<') equals -v (R10).
 * RMC: REJECTED iff some delta != 0 in [-S,S]^2 has a strictly smaller mean
 *      rc(x, -v+delta) than delta = 0 (R11), else ACCEPTED.
 * Reads entries with status CANDIDATE or ACCEPTED in rows [y_begin, y_end),
 * writes ACCEPTED / REJECTED into io->status; never touches alpha, beta, err,
 * count.  Buffers must hold rows [y_begin - 2S - K, y_end + 2S + K) clipped.
 * eval_count (nullable, device) += (2S+1)^2 per checked entry (R17).
 * workspace: QS_RME needs qs_workspace_size() bytes; QS_RMC none (may be NULL).
 * ------------------------------------------------------------------------- */
int qs_reverse_check(int32_t mode, const uint8_t *cur, const uint8_t *cur_mask, int64_t cur_pitch,
                     const void *ref, int64_t ref_pitch, const qs_roi *roi, const qs_me_params *p,
                     qs_field *io, unsigned long long *eval_count, void *workspace, size_t workspace_bytes,
                     void *stream);

/* ---------------------------------------------------------------------------
 * qs_frmc -- fast reverse motion check (§3.1.1: "we test only
 * motions in the set {-7,-3,-1,0,1,3,7} for both spatial dimensions ... If the
 * green arrow has the lowest cost, the motion is accepted. If any of the red
 * arrows has the lowest cost, the motion is rejected.").
 * As RMC with delta in offsets x offsets.  offsets is a HOST array (1..15
 * entries, must contain 0, |o| <= 32).  Buffers must hold rows
 * [y_begin - max|o| - K, y_end + max|o| + K) clipped.
 * eval_count += n_offsets^2 per checked entry.
 * ------------------------------------------------------------------------- */
int qs_frmc(const uint8_t *cur, const uint8_t *cur_mask, int64_t cur_pitch,
            const void *ref, int64_t ref_pitch, const qs_roi *roi, const qs_me_params *p,
            const int8_t *offsets, int32_t n_offsets, qs_field *io,
            unsigned long long *eval_count, void *stream);

/* ---------------------------------------------------------------------------
 * qs_nnc -- nearest-neighbour check (§3.1.2, Eq. (1)):
 * component-wise 3x3 median over VALID entries (status >= CANDIDATE, whatever
 * the accept state; in-frame window, centre included, lower median; R14), then
 * an entry with status CANDIDATE or ACCEPTED is REJECTED iff some in-frame valid
 * 4-neighbour has |a~(p)-a~(nb)| + |b~(p)-b~(nb)| > threshold, else ACCEPTED
 * (R15).  Rows [y_begin, y_end) are decided; the field buffer must hold rows
 * [y_begin-2, y_end+2) clipped (reads only alpha, beta, status; writes status).
 * In-place is safe: the filter reads a snapshot taken inside the kernel.
 * ------------------------------------------------------------------------- */
int qs_nnc(qs_field *io, const qs_roi *roi, int32_t threshold, void *stream);

/* qs_nnc with the reading chosen: mode QS_NNC_CENTRE (= qs_nnc) or QS_NNC_PAIRS (the valid in-frame
 * filtered 4-neighbours compared with each other, every unordered pair; REJECTED iff some pair differs
 * by more than threshold; fewer than two tested neighbours -> ACCEPTED).  Other modes QS_EINVAL. */
int qs_nnc_mode(qs_field *io, const qs_roi *roi, int32_t threshold, int32_t mode, void *stream);

/* ---------------------------------------------------------------------------
 * qs_project -- projection PR (§2.2: "If a measurement is
 * available at the corresponding position in the past frame, it is projected to
 * the current frame ... In case projections from more than one past frame are
 * available, these are averaged."; R18).
 * For each ACCEPTED p in rows [y_begin, y_end): q = p+v; if q is in the frame
 * and past_mask(q) == 1: sum(p) += past_val(q), cnt(p) += 1.  ACCUMULATES into
 * caller-zeroed sum (uint32) / cnt (uint8) planes [rows][acc_pitch elements],
 * so successive calls for d = 1, 2, 3 average across references.  past_* must
 * hold rows [y_begin - S, y_end + S) clipped (|alpha| <= S).  The call has no S
 * to validate that against: an ACCEPTED entry whose q = p+v lies outside the
 * past buffers' row window [buf_y0, buf_y0 + buf_rows) is NOT projected (no
 * error is returned), so a caller passing too few past rows gets smaller
 * sum / cnt for those entries.
 * ------------------------------------------------------------------------- */
int qs_project(const qs_field *f, const uint8_t *past_val, const uint8_t *past_mask, int64_t past_pitch,
               const qs_roi *roi, uint32_t *sum, uint8_t *cnt, int64_t acc_pitch, void *stream);

/* ---------------------------------------------------------------------------
 * Launch timing (the profiling subsystem; SURVEY.md §5 "CUDA events per stage").
 * While enabled, every kernel launched by the entry points above is bracketed
 * by two CUDA events recorded on its own stream.  qs_profile_read synchronises
 * the recorded events and returns the summed device time and the number of
 * bracketed launches of one kernel ("me_box", "epilogue", "finalize", "nnc",
 * "revgrid", "rme_decide", "project", "certify") or of all of them ("*"); one
 * bracket can hold several grids (certify: scan + fix; me_box on float
 * references: the border grid and the interior grid).  qs_profile_reset drops
 * the records.
 * Process-global; calls from several threads are serialised internally.
 * ------------------------------------------------------------------------- */
int qs_profile_enable(int32_t on);
int qs_profile_read(const char *kernel, double *total_ms, int64_t *launches);
int qs_profile_reset(void);

/* ---------------------------------------------------------------------------
 * qs_certify_stats -- float references only: the number of
 * outputs (forward targets and reverse positions) whose approximate argmin could not be certified
 * and were recomputed exactly in the definition's arithmetic, summed over every call on the current
 * device since the last reset.  Synchronises the device.  reset != 0 zeroes the counter after
 * reading it.  QS_EINVAL for a NULL pointer, QS_ECUDA if the device access fails.
 * ------------------------------------------------------------------------- */
int qs_certify_stats(int64_t *rechecked, int32_t reset);

/* Thread-local message describing the last non-QS_OK return on this thread. */
const char *qs_last_error(void);

/* Library version / build string (e.g. "libqs 0.1 sm_100a"). */
const char *qs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QS_H_ */

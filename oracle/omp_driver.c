/*
 * omp_driver.c -- OpenMP driver over target rows for the oracle (TEST INFRASTRUCTURE ONLY;
 * same import rules as oracle.c).  It adds no arithmetic: every row is one call of the untouched,
 * single-threaded definitions in oracle.c on the row range [y, y+1), so the result is the
 * sequential oracle's for any thread count (the definitions write only their own rows' entries).
 * Used to verify full frames at config-4/5 sizes and for the all-core oracle timing (SURVEY.md
 * §8(d.5) mode 2: "OpenMP over target rows on all host cores").  Built with -fopenmp into
 * liboracle_omp.so next to liboracle.so.
 */
#include <stdint.h>
#include <stddef.h>
#include <omp.h>

typedef struct {
    int32_t W, H, Kh, Kw, S, min_support, ssd, ref_mode;
} or_params;   /* layout of oracle.c's or_params */

int or_me_search(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                 int32_t y_begin, int32_t y_end,
                 int8_t *alpha, int8_t *beta, void *err, uint8_t *count, uint8_t *status);
int or_frmc(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
            const int32_t *offsets, int32_t n_offsets, int32_t y_begin, int32_t y_end,
            const int8_t *alpha, const int8_t *beta, const void *err, const uint8_t *count,
            uint8_t *status, uint64_t *evals, int32_t verify_p4);
int or_rmc(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
           int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
           const void *err, const uint8_t *count, uint8_t *status, uint64_t *evals, int32_t verify_p4);
int or_rme(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
           int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
           const void *err, const uint8_t *count, uint8_t *status, uint64_t *evals);

int or_threads_available(void) { return omp_get_max_threads(); }

int or_me_search_omp(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                     int32_t y_begin, int32_t y_end, int8_t *alpha, int8_t *beta, void *err,
                     uint8_t *count, uint8_t *status, int32_t threads) {
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(| : bad)
    for (int y = y_begin; y < y_end; ++y)
        bad |= or_me_search(P, cur, mask, ref, y, y + 1, alpha, beta, err, count, status) != 0;
    return bad ? -1 : 0;
}

int or_frmc_omp(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
                const int32_t *offsets, int32_t n_offsets, int32_t y_begin, int32_t y_end,
                const int8_t *alpha, const int8_t *beta, const void *err, const uint8_t *count,
                uint8_t *status, uint64_t *evals, int32_t verify_p4, int32_t threads) {
    int bad = 0;
    uint64_t ev = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(| : bad) reduction(+ : ev)
    for (int y = y_begin; y < y_end; ++y) {
        uint64_t e = 0;
        bad |= or_frmc(P, cur, mask, ref, offsets, n_offsets, y, y + 1, alpha, beta, err, count, status, &e,
                       verify_p4) != 0;
        ev += e;
    }
    if (evals) *evals += ev;
    return bad ? -1 : 0;
}

int or_rmc_omp(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
               int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
               const void *err, const uint8_t *count, uint8_t *status, uint64_t *evals, int32_t verify_p4,
               int32_t threads) {
    int bad = 0;
    uint64_t ev = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(| : bad) reduction(+ : ev)
    for (int y = y_begin; y < y_end; ++y) {
        uint64_t e = 0;
        bad |= or_rmc(P, cur, mask, ref, y, y + 1, alpha, beta, err, count, status, &e, verify_p4) != 0;
        ev += e;
    }
    if (evals) *evals += ev;
    return bad ? -1 : 0;
}

int or_rme_omp(const or_params *P, const uint8_t *cur, const uint8_t *mask, const void *ref,
               int32_t y_begin, int32_t y_end, const int8_t *alpha, const int8_t *beta,
               const void *err, const uint8_t *count, uint8_t *status, uint64_t *evals, int32_t threads) {
    int bad = 0;
    uint64_t ev = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(| : bad) reduction(+ : ev)
    for (int y = y_begin; y < y_end; ++y) {
        uint64_t e = 0;
        bad |= or_rme(P, cur, mask, ref, y, y + 1, alpha, beta, err, count, status, &e) != 0;
        ev += e;
    }
    if (evals) *evals += ev;
    return bad ? -1 : 0;
}

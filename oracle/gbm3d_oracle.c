/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU reference for
 * the G-BM3D block-matching stage (arXiv 2103.10765, section II and III-B).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code, header, table or helper with the CUDA
 * path in paper_2103_10765_b200/ (DESIGN.md "Oracle").
 *
 * What it computes is the plain definition, not the paper's fast procedure: the paper
 * states the fast scheme "does not change the design of the block matching, but only
 * the computational procedure", so the definition is the oracle:
 *
 *   step 1  reference grid R = {0, s, 2s, ... <= L-P} U {L-P}   (tiles at (pN,qN),
 *           PAPER.md:156; appended last position = DESIGN.md reading R3)
 *   step 2  window C(rho) = {c : |c-rho|_inf <= r, 0 <= c <= (H-P, W-P)} (local search,
 *           PAPER.md:75,121; clamped, no wrap = reading R2)
 *   step 3  d(rho,c) = sum_{i,j<P} (Z[ry+i][rx+j] - Z[cy+i][cx+j])^2   (Eq. (1)),
 *           accumulated in int64 and required to fit int32 (reading R10)
 *   step 4  L(rho) = sorted{(d, idx) : c in C(rho) \ {rho}, d < tau}  (strict <, PAPER.md:73;
 *           key (d, idx = cy*W+cx) = reading R5)
 *   step 5  out = [(idx(rho), 0)] + L[:K-1]; n_valid = len(out); pad (idx(rho), -1)
 *           (S^K_pq includes self, "exactly 15 matches" for K=16, PAPER.md:134,158;
 *           "padded with the reference block", PAPER.md:134 = readings R4, R7)
 *
 * Parity pins (tests/test_oracle.py): exhaustive pure-Python enumeration, scipy cdist,
 * Eq. (2) in exact integers, constant/periodic closed forms, symmetry,
 * completeness, tau/K/r special cases, hand-worked golden fixtures.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_ARG (-1)
#define ORACLE_ERR_RANGE (-2)
#define ORACLE_ERR_NOMEM (-5)

typedef struct {
    int64_t d;
    int64_t idx;
} oracle_cand;

/* step 4 ordering: lexicographic on (d, idx) -- reading R5 */
static int oracle_cmp(const void* pa, const void* pb) {
    const oracle_cand* a = (const oracle_cand*)pa;
    const oracle_cand* b = (const oracle_cand*)pb;
    if (a->d != b->d) return a->d < b->d ? -1 : 1;
    if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
    return 0;
}

/* step 1: positions 0, s, 2s, ... <= L-P, then L-P if it is not already there.
 * Returns the count; writes positions to out when out != NULL. */
int oracle_grid(int L, int P, int s, int* out) {
    if (L < P || P < 1 || s < 1) return 0;
    int n = 0, last = L - P, p;
    for (p = 0; p <= last; p += s) {
        if (out) out[n] = p;
        n++;
    }
    if ((last % s) != 0) {
        if (out) out[n] = last;
        n++;
    }
    return n;
}

/* step 3: Eq. (1) written out, two loops over the P x P block, int64 accumulation. */
int64_t oracle_patch_ssd(const int16_t* img, int W, int ay, int ax, int by, int bx, int P) {
    int64_t acc = 0;
    for (int i = 0; i < P; i++) {
        for (int j = 0; j < P; j++) {
            int64_t diff = (int64_t)img[(int64_t)(ay + i) * W + (ax + j)] -
                           (int64_t)img[(int64_t)(by + i) * W + (bx + j)];
            acc += diff * diff;
        }
    }
    return acc;
}

/*
 * The whole stage for one image.  Outputs are int32 [Ry][Rx][K] (idx, dist) and
 * [Ry][Rx] (n_valid, nullable).  tau < 0 means "no threshold".
 * Returns ORACLE_ERR_RANGE if any distance exceeds INT32_MAX (outputs then undefined).
 */
int oracle_block_match(const int16_t* img, int H, int W, int P, int s, int r, int K,
                       int64_t tau, int32_t* idx_out, int32_t* dist_out, int32_t* nvalid_out,
                       int nthreads) {
    if (!img || !idx_out || !dist_out || H < P || W < P || P < 1 || s < 1 || r < 0 || K < 1)
        return ORACLE_ERR_ARG;
    int Ry = oracle_grid(H, P, s, NULL), Rx = oracle_grid(W, P, s, NULL);
    int* gy = (int*)malloc(sizeof(int) * (size_t)Ry);
    int* gx = (int*)malloc(sizeof(int) * (size_t)Rx);
    if (!gy || !gx) {
        free(gy);
        free(gx);
        return ORACLE_ERR_NOMEM;
    }
    oracle_grid(H, P, s, gy);
    oracle_grid(W, P, s, gx);
    const int side = 2 * r + 1;
    const int64_t max_cands = (int64_t)(side < H ? side : H) * (int64_t)(side < W ? side : W);
    int status = ORACLE_OK;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

#pragma omp parallel
    {
        oracle_cand* cands = (oracle_cand*)malloc(sizeof(oracle_cand) * (size_t)max_cands);
        if (!cands) {
#pragma omp atomic write
            status = ORACLE_ERR_NOMEM;
        }
#pragma omp for schedule(dynamic)
        for (int py = 0; py < Ry; py++) {
            if (!cands) continue;
            for (int px = 0; px < Rx; px++) {
                const int ry = gy[py], rx = gx[px];
                const int64_t self_idx = (int64_t)ry * W + rx;
                /* step 2: clamped window */
                int cy0 = ry - r < 0 ? 0 : ry - r;
                int cy1 = ry + r > H - P ? H - P : ry + r;
                int cx0 = rx - r < 0 ? 0 : rx - r;
                int cx1 = rx + r > W - P ? W - P : rx + r;
                int64_t n = 0;
                for (int cy = cy0; cy <= cy1; cy++) {
                    for (int cx = cx0; cx <= cx1; cx++) {
                        if (cy == ry && cx == rx) continue; /* self goes to slot 0 (step 5) */
                        int64_t d = oracle_patch_ssd(img, W, ry, rx, cy, cx, P);
                        if (d > INT32_MAX) {
#pragma omp atomic write
                            status = ORACLE_ERR_RANGE;
                        }
                        if (tau >= 0 && !(d < tau)) continue; /* strict, Eq. (1) */
                        cands[n].d = d;
                        cands[n].idx = (int64_t)cy * W + cx;
                        n++;
                    }
                }
                qsort(cands, (size_t)n, sizeof(oracle_cand), oracle_cmp);
                /* step 5 */
                const int64_t base = ((int64_t)py * Rx + px) * K;
                idx_out[base] = (int32_t)self_idx;
                dist_out[base] = 0;
                int nv = 1;
                for (int k = 1; k < K; k++) {
                    if (k - 1 < n) {
                        idx_out[base + k] = (int32_t)cands[k - 1].idx;
                        dist_out[base + k] = (int32_t)cands[k - 1].d;
                        nv++;
                    } else {
                        idx_out[base + k] = (int32_t)self_idx;
                        dist_out[base + k] = -1;
                    }
                }
                if (nvalid_out) nvalid_out[(int64_t)py * Rx + px] = nv;
            }
        }
        free(cands);
    }
    free(gy);
    free(gx);
    return status;
}

/*
 * The same definition (steps 2-5) for an explicit list of reference grid cells (py[i], px[i]),
 * used to check full-size GPU runs on sampled references.  Outputs are [n][K] and [n].
 */
int oracle_block_match_refs(const int16_t* img, int H, int W, int P, int s, int r, int K,
                            int64_t tau, const int32_t* py_list, const int32_t* px_list, int n,
                            int32_t* idx_out, int32_t* dist_out, int32_t* nvalid_out,
                            int nthreads) {
    if (!img || !idx_out || !dist_out || !py_list || !px_list || n < 0 || H < P || W < P ||
        P < 1 || s < 1 || r < 0 || K < 1)
        return ORACLE_ERR_ARG;
    int Ry = oracle_grid(H, P, s, NULL), Rx = oracle_grid(W, P, s, NULL);
    int* gy = (int*)malloc(sizeof(int) * (size_t)Ry);
    int* gx = (int*)malloc(sizeof(int) * (size_t)Rx);
    if (!gy || !gx) {
        free(gy);
        free(gx);
        return ORACLE_ERR_NOMEM;
    }
    oracle_grid(H, P, s, gy);
    oracle_grid(W, P, s, gx);
    int status = ORACLE_OK;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic)
    for (int t = 0; t < n; t++) {
        if (py_list[t] < 0 || py_list[t] >= Ry || px_list[t] < 0 || px_list[t] >= Rx) {
#pragma omp atomic write
            status = ORACLE_ERR_ARG;
            continue;
        }
        /* one-reference view: call the whole-image routine on a 1x1 grid is not possible, so
           steps 2-5 are written out again here, literally as above */
        const int ry = gy[py_list[t]], rx = gx[px_list[t]];
        const int64_t self_idx = (int64_t)ry * W + rx;
        int cy0 = ry - r < 0 ? 0 : ry - r;
        int cy1 = ry + r > H - P ? H - P : ry + r;
        int cx0 = rx - r < 0 ? 0 : rx - r;
        int cx1 = rx + r > W - P ? W - P : rx + r;
        oracle_cand* cands =
            (oracle_cand*)malloc(sizeof(oracle_cand) * (size_t)((cy1 - cy0 + 1) * (cx1 - cx0 + 1)));
        if (!cands) {
#pragma omp atomic write
            status = ORACLE_ERR_NOMEM;
            continue;
        }
        int64_t m = 0;
        for (int cy = cy0; cy <= cy1; cy++) {
            for (int cx = cx0; cx <= cx1; cx++) {
                if (cy == ry && cx == rx) continue;
                int64_t d = oracle_patch_ssd(img, W, ry, rx, cy, cx, P);
                if (d > INT32_MAX) {
#pragma omp atomic write
                    status = ORACLE_ERR_RANGE;
                }
                if (tau >= 0 && !(d < tau)) continue;
                cands[m].d = d;
                cands[m].idx = (int64_t)cy * W + cx;
                m++;
            }
        }
        qsort(cands, (size_t)m, sizeof(oracle_cand), oracle_cmp);
        const int64_t base = (int64_t)t * K;
        idx_out[base] = (int32_t)self_idx;
        dist_out[base] = 0;
        int nv = 1;
        for (int k = 1; k < K; k++) {
            if (k - 1 < m) {
                idx_out[base + k] = (int32_t)cands[k - 1].idx;
                dist_out[base + k] = (int32_t)cands[k - 1].d;
                nv++;
            } else {
                idx_out[base + k] = (int32_t)self_idx;
                dist_out[base + k] = -1;
            }
        }
        if (nvalid_out) nvalid_out[t] = nv;
        free(cands);
    }
    free(gy);
    free(gx);
    return status;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * lp_oracle.c -- CPU restatement of the reference's label-propagation path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
 * leg load it (as the checker / the timed CPU arm), never as the measured or
 * shipped path.
 *
 * Pinned against the reference (see tests/golden/make_golden.py, which runs
 * the numba reference from /root/reference and stores its outputs):
 *   - or_rak() with batches == n and tie OR_TIE_XORSHIFT / OR_TIE_SCAN_FIRST
 *     reproduces rak._rak_seq bit for bit (labels and iteration count);
 *   - or_shuffled_indices() reproduces prng.shuffled_indices;
 *   - or_copra() reproduces copra._copra_seq; or_slpa() reproduces
 *     slpa._slpa_seq + _project.
 *
 * Reference anchors (paths under /root/reference/pkg/src/labelprop/):
 *   prng.py:29-36   xs32_next          -> or_xs32_next
 *   prng.py:39-44   draw_bounded       -> or_draw
 *   prng.py:47-63   mix_seed           -> or_mix_seed
 *   prng.py:82-94   shuffled_indices   -> or_shuffled_indices
 *   rak.py:57-84    _pick_from_tally   -> pick_from_tally
 *   rak.py:87-116   _rak_seq           -> or_rak (batches == n)
 *   rak.py:119-158  _rak_par           -> or_rak_par (OpenMP port)
 *   copra.py:53-121 _select_labels, _best_of_row
 *   copra.py:124-176 _copra_seq        -> or_copra
 *   slpa.py:51-111  _modal_label, _listen, _slpa_seq -> or_slpa
 *   slpa.py:147-150 _project
 *
 * Generalisation used to pin the GPU engine: the batched schedule.  The
 * visit order is cut into B contiguous batches of ceil(n/B) vertices; every
 * member of a batch is computed from the labels as they stood at the start
 * of that batch, then the batch commits.  B == n is the reference's
 * asynchronous in-place sweep; B == 1 is the synchronous (Jacobi) sweep.
 *
 * Tie rules:
 *   OR_TIE_SCAN_FIRST  strict: first maximum in CSR scan order (rak.py:61-70)
 *   OR_TIE_XORSHIFT    non-strict, reference RNG stream: the j-th tie in
 *                      first-touch order, j = xorshift draw % ties (rak.py:71-83)
 *   OR_TIE_RANDOM      non-strict, counter RNG (the GPU rule): among the
 *                      maximum-weight labels pick the one with the largest
 *                      or_tie_hash(seed, sweep, vertex, label); equal hashes
 *                      fall back to first-touch order
 *   OR_TIE_MIN_LABEL   smallest label id among the maxima (BASELINE config 0
 *                      wording; not the reference's rule)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_TIE_SCAN_FIRST 0
#define OR_TIE_RANDOM 1
#define OR_TIE_MIN_LABEL 2
#define OR_TIE_XORSHIFT 3

#define OR_ZERO_SEED 2463534242u /* prng.py:26 */
#define OR_ORDER_STREAM 0x4F524452u /* prng.py:79 */

uint32_t or_xs32_next(uint32_t x) {
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    return x;
}

static inline uint32_t or_draw(uint32_t* state, uint32_t bound) {
    *state = or_xs32_next(*state);
    return *state % bound;
}

static inline uint32_t fmix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x85EBCA6Bu;
    x ^= x >> 13;
    x *= 0xC2B2AE35u;
    x ^= x >> 16;
    return x;
}

uint32_t or_mix_seed(uint32_t seed, uint32_t k) {
    uint32_t x = fmix32(seed + k * 0x9E3779B9u);
    return x ? x : OR_ZERO_SEED;
}

void or_shuffled_indices(int64_t n, uint32_t seed, int64_t* order) {
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    uint32_t st = or_mix_seed(seed, OR_ORDER_STREAM);
    for (int64_t i = n - 1; i > 0; --i) {
        int64_t j = (int64_t)or_draw(&st, (uint32_t)(i + 1));
        int64_t t = order[i];
        order[i] = order[j];
        order[j] = t;
    }
}

/* Counter RNG for non-strict ties, shared definition with the CUDA engine
 * (DESIGN.md "tie rules"): a murmur3-fmix32 chain over (seed, sweep,
 * vertex, label). */
uint32_t or_tie_hash(uint32_t seed, uint32_t sweep, uint32_t vertex, uint32_t label) {
    uint32_t h = fmix32(seed ^ (sweep * 0x9E3779B9u + 0x7F4A7C15u));
    h = fmix32(h ^ (vertex * 0x85EBCA6Bu + 0x68E31DA4u));
    h = fmix32(h ^ (label * 0xC2B2AE35u + 0xB5297A4Du));
    return h;
}

/* Scratch shared by the tally-based kernels (dense tally + touched list,
 * like rak.py:175-176). */
typedef struct {
    double* tally;
    int64_t* touched;
} scratch_t;

static int scratch_init(scratch_t* s, int64_t n) {
    s->tally = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    s->touched = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    return (s->tally && s->touched) ? 0 : -1;
}
static void scratch_free(scratch_t* s) {
    free(s->tally);
    free(s->touched);
}

/* rak.py:57-84 generalised over the tie rules. */
static int64_t pick_from_tally(const int64_t* touched, const double* tally, int64_t count, int tie,
                               uint32_t* xs_state, uint32_t seed, uint32_t sweep, uint32_t vertex) {
    double best_w = -1.0;
    int64_t best = -1;
    for (int64_t i = 0; i < count; ++i) {
        double w = tally[touched[i]];
        if (w > best_w) {
            best_w = w;
            best = touched[i];
        }
    }
    if (tie == OR_TIE_SCAN_FIRST || count == 1) return best;
    if (tie == OR_TIE_MIN_LABEL) {
        for (int64_t i = 0; i < count; ++i)
            if (tally[touched[i]] == best_w && touched[i] < best) best = touched[i];
        return best;
    }
    if (tie == OR_TIE_RANDOM) {
        uint32_t best_h = 0;
        int have = 0;
        for (int64_t i = 0; i < count; ++i) {
            if (tally[touched[i]] != best_w) continue;
            uint32_t h = or_tie_hash(seed, sweep, vertex, (uint32_t)touched[i]);
            if (!have || h > best_h) {
                have = 1;
                best_h = h;
                best = touched[i];
            }
        }
        return best;
    }
    /* OR_TIE_XORSHIFT: the reference's rule */
    int64_t ties = 0;
    for (int64_t i = 0; i < count; ++i)
        if (tally[touched[i]] == best_w) ++ties;
    if (ties == 1) return best;
    uint32_t j = or_draw(xs_state, (uint32_t)ties);
    for (int64_t i = 0; i < count; ++i) {
        if (tally[touched[i]] == best_w) {
            if (j == 0) return touched[i];
            --j;
        }
    }
    return best;
}

/* Tally of vertex v's arcs over the label array `lab` (rak.py:99-105);
 * weights NULL means unit weights. */
static int64_t tally_row(const int64_t* off, const int64_t* nbr, const double* w, const int64_t* lab,
                         int64_t v, scratch_t* s) {
    int64_t count = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int64_t l = lab[nbr[e]];
        if (s->tally[l] == 0.0) s->touched[count++] = l;
        s->tally[l] += w ? w[e] : 1.0;
    }
    return count;
}

static void untally(scratch_t* s, int64_t count) {
    for (int64_t i = 0; i < count; ++i) s->tally[s->touched[i]] = 0.0;
}

/*
 * Batched RAK.  labels: in = initial labels (the reference uses arange(n)),
 * out = final labels.  Returns the iteration count (rak.py:94-95 semantics:
 * the sweep that meets the tolerance is counted), or -1 on allocation
 * failure.  changed_per_iter[it] and labels_per_iter[it*n ...] are filled
 * when non-NULL (arrays of max_it entries / max_it*n labels).
 */
int or_rak(int64_t n, const int64_t* off, const int64_t* nbr, const double* w, const int64_t* order,
           int64_t batches, int tie, uint32_t seed, double tol, int max_it, int64_t* labels,
           int64_t* changed_per_iter, int64_t* labels_per_iter) {
    if (n == 0) return 0;
    if (batches <= 0 || batches > n) batches = n;
    int64_t bs = (n + batches - 1) / batches;
    scratch_t s;
    if (scratch_init(&s, n)) return -1;
    int64_t* fresh = (int64_t*)malloc((size_t)bs * sizeof(int64_t));
    if (!fresh) {
        scratch_free(&s);
        return -1;
    }
    uint32_t xs = or_mix_seed(seed, 0); /* worker_states(seed, 1)[0], prng.py:66-74 */
    int it = 0;
    while (it < max_it) {
        ++it;
        int64_t changed = 0;
        for (int64_t b0 = 0; b0 < n; b0 += bs) {
            int64_t b1 = b0 + bs < n ? b0 + bs : n;
            /* every member reads the labels as they stand at batch start */
            for (int64_t i = b0; i < b1; ++i) {
                int64_t v = order[i];
                int64_t count = tally_row(off, nbr, w, labels, v, &s);
                if (count == 0) { /* no arcs: label cannot move (rak.py:106-107) */
                    fresh[i - b0] = labels[v];
                    continue;
                }
                fresh[i - b0] = pick_from_tally(s.touched, s.tally, count, tie, &xs, seed,
                                                (uint32_t)it, (uint32_t)v);
                untally(&s, count);
            }
            for (int64_t i = b0; i < b1; ++i) {
                int64_t v = order[i];
                if (fresh[i - b0] != labels[v]) {
                    labels[v] = fresh[i - b0];
                    ++changed;
                }
            }
        }
        if (changed_per_iter) changed_per_iter[it - 1] = changed;
        if (labels_per_iter) memcpy(labels_per_iter + (int64_t)(it - 1) * n, labels, (size_t)n * 8);
        if ((double)changed <= tol * (double)n) break; /* rak.py:114-115 */
    }
    free(fresh);
    scratch_free(&s);
    return it;
}

/*
 * OpenMP port of rak._rak_par (rak.py:119-158): the permutation is handed
 * out in chunks of `chunk` vertices (dynamic schedule, SPEC "dynamic chunks
 * of 1024"), each thread owns a dense tally row and xorshift state
 * worker_states(seed, W)[tid], labels are read and written in place with
 * relaxed word-sized atomics (the reference's benign races, SPEC.md
 * "Concurrency Model").  Non-deterministic for threads > 1, like the
 * reference.  tie: OR_TIE_SCAN_FIRST (strict) or OR_TIE_XORSHIFT.
 * This is the CPU baseline arm of bench.py.
 */
int or_rak_par(int64_t n, const int64_t* off, const int64_t* nbr, const double* w, const int64_t* order,
               int tie, uint32_t seed, double tol, int max_it, int threads, int64_t chunk,
               int64_t* labels) {
    if (n == 0) return 0;
    if (threads < 1) threads = 1;
    if (chunk < 1) chunk = 1024;
    int64_t n_chunks = (n + chunk - 1) / chunk;
    int nt = threads;
    double** tallies = (double**)calloc((size_t)nt, sizeof(double*));
    int64_t** touches = (int64_t**)calloc((size_t)nt, sizeof(int64_t*));
    uint32_t* states = (uint32_t*)calloc((size_t)nt * 16, sizeof(uint32_t)); /* padded */
    int fail = !tallies || !touches || !states;
    for (int t = 0; t < nt && !fail; ++t) {
        tallies[t] = (double*)calloc((size_t)n + 8, sizeof(double));
        touches[t] = (int64_t*)malloc(((size_t)n + 8) * sizeof(int64_t));
        fail |= !tallies[t] || !touches[t];
        if (states) states[t * 16] = or_mix_seed(seed, (uint32_t)t);
    }
    int it = 0;
    if (!fail) {
        while (it < max_it) {
            ++it;
            int64_t changed = 0;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1) reduction(+ : changed)
            for (int64_t c = 0; c < n_chunks; ++c) {
                int tid = 0;
#ifdef _OPENMP
                tid = omp_get_thread_num();
#endif
                double* tally = tallies[tid];
                int64_t* touched = touches[tid];
                int64_t hi = (c + 1) * chunk < n ? (c + 1) * chunk : n;
                for (int64_t i = c * chunk; i < hi; ++i) {
                    int64_t v = order[i];
                    int64_t count = 0;
                    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
                        int64_t l = __atomic_load_n(&labels[nbr[e]], __ATOMIC_RELAXED);
                        if (tally[l] == 0.0) touched[count++] = l;
                        tally[l] += w ? w[e] : 1.0;
                    }
                    if (count == 0) continue;
                    int64_t best = pick_from_tally(touched, tally, count, tie, &states[tid * 16], seed,
                                                   (uint32_t)it, (uint32_t)v);
                    for (int64_t k = 0; k < count; ++k) tally[touched[k]] = 0.0;
                    if (best != __atomic_load_n(&labels[v], __ATOMIC_RELAXED)) {
                        __atomic_store_n(&labels[v], best, __ATOMIC_RELAXED);
                        ++changed;
                    }
                }
            }
            if ((double)changed <= tol * (double)n) break;
        }
    }
    for (int t = 0; t < nt && tallies && touches; ++t) {
        free(tallies[t]);
        free(touches[t]);
    }
    free(tallies);
    free(touches);
    free(states);
    return fail ? -1 : it;
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------- */
/* COPRA (copra.py)                                                       */
/* ---------------------------------------------------------------------- */

/* copra.py:53-108 _select_labels; returns k and fills out_l/out_b sorted
 * by label id.  rng: reference xorshift stream (tie == OR_TIE_XORSHIFT) or
 * the counter rule (tie == OR_TIE_RANDOM) for the GPU batched schedule. */
static int64_t select_labels(const int64_t* touched, const double* tally, int64_t count, int64_t max_labels,
                             int tie, uint32_t* xs, uint32_t seed, uint32_t sweep, uint32_t vertex,
                             int64_t* out_l, double* out_b) {
    double total = 0.0;
    for (int64_t i = 0; i < count; ++i) total += tally[touched[i]];
    int64_t k = 0;
    double kept = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        int64_t lab = touched[i];
        double w = tally[lab];
        if (w * (double)max_labels >= total && k < max_labels) {
            out_l[k] = lab;
            out_b[k] = w;
            kept += w;
            ++k;
        }
    }
    if (k == 0) {
        double best_w = -1.0;
        for (int64_t i = 0; i < count; ++i)
            if (tally[touched[i]] > best_w) best_w = tally[touched[i]];
        if (tie == OR_TIE_RANDOM) {
            uint32_t bh = 0;
            int have = 0;
            int64_t best = -1;
            for (int64_t i = 0; i < count; ++i) {
                if (tally[touched[i]] != best_w) continue;
                uint32_t h = or_tie_hash(seed, sweep, vertex, (uint32_t)touched[i]);
                if (!have || h > bh) {
                    have = 1;
                    bh = h;
                    best = touched[i];
                }
            }
            out_l[0] = best;
            out_b[0] = 1.0;
            return 1;
        }
        int64_t ties = 0;
        for (int64_t i = 0; i < count; ++i)
            if (tally[touched[i]] == best_w) ++ties;
        uint32_t j = 0;
        if (ties > 1) j = or_draw(xs, (uint32_t)ties);
        for (int64_t i = 0; i < count; ++i) {
            if (tally[touched[i]] == best_w) {
                if (j == 0) {
                    out_l[0] = touched[i];
                    out_b[0] = 1.0;
                    return 1;
                }
                --j;
            }
        }
        return 1;
    }
    double inv = 1.0 / kept;
    for (int64_t i = 0; i < k; ++i) out_b[i] *= inv;
    for (int64_t i = 1; i < k; ++i) {
        int64_t lab = out_l[i];
        double b = out_b[i];
        int64_t j = i - 1;
        while (j >= 0 && out_l[j] > lab) {
            out_l[j + 1] = out_l[j];
            out_b[j + 1] = out_b[j];
            --j;
        }
        out_l[j + 1] = lab;
        out_b[j + 1] = b;
    }
    return k;
}

/* copra.py:111-121 */
static int64_t best_of_row(const int64_t* l, const double* b, int64_t k) {
    int64_t best = l[0];
    double bb = b[0];
    for (int64_t j = 1; j < k; ++j)
        if (b[j] > bb) {
            bb = b[j];
            best = l[j];
        }
    return best;
}

/*
 * COPRA with the batched schedule over index order (copra.py:134 visits
 * v = 0..n-1; batches == n reproduces _copra_seq).  labs/bels are n x L
 * row-major, sizes n, best n; all in/out (caller initialises them as
 * copra.py:254-258).  Returns iterations.
 */
int or_copra(int64_t n, const int64_t* off, const int64_t* nbr, const double* w, int64_t max_labels,
             int64_t batches, int tie, uint32_t seed, double tol, int max_it, int64_t* labs, double* bels,
             int64_t* sizes, int64_t* best) {
    if (n == 0) return 0;
    if (batches <= 0 || batches > n) batches = n;
    int64_t bs = (n + batches - 1) / batches;
    int64_t L = max_labels;
    scratch_t s;
    if (scratch_init(&s, n)) return -1;
    int64_t* nl = (int64_t*)malloc((size_t)(bs * L) * sizeof(int64_t));
    double* nb = (double*)malloc((size_t)(bs * L) * sizeof(double));
    int64_t* ns = (int64_t*)malloc((size_t)bs * sizeof(int64_t));
    int64_t* nbest = (int64_t*)malloc((size_t)bs * sizeof(int64_t));
    if (!nl || !nb || !ns || !nbest) return -1;
    uint32_t xs = or_mix_seed(seed, 0);
    int it = 0;
    while (it < max_it) {
        ++it;
        int64_t changed = 0;
        for (int64_t b0 = 0; b0 < n; b0 += bs) {
            int64_t b1 = b0 + bs < n ? b0 + bs : n;
            for (int64_t v = b0; v < b1; ++v) {
                int64_t count = 0;
                for (int64_t e = off[v]; e < off[v + 1]; ++e) {
                    int64_t u = nbr[e];
                    if (u == v) continue; /* copra.py:137-139 */
                    double we = w ? w[e] : 1.0;
                    for (int64_t j = 0; j < sizes[u]; ++j) {
                        int64_t lab = labs[u * L + j];
                        if (s.tally[lab] == 0.0) s.touched[count++] = lab;
                        s.tally[lab] += bels[u * L + j] * we;
                    }
                }
                int64_t r = v - b0;
                if (count == 0) { /* copra.py:147-151 */
                    nl[r * L] = v;
                    nb[r * L] = 1.0;
                    ns[r] = 1;
                    nbest[r] = v;
                } else {
                    ns[r] = select_labels(s.touched, s.tally, count, L, tie, &xs, seed, (uint32_t)it,
                                          (uint32_t)v, nl + r * L, nb + r * L);
                    untally(&s, count);
                    nbest[r] = best_of_row(nl + r * L, nb + r * L, ns[r]);
                }
            }
            for (int64_t v = b0; v < b1; ++v) {
                int64_t r = v - b0;
                sizes[v] = ns[r];
                for (int64_t j = 0; j < ns[r]; ++j) {
                    labs[v * L + j] = nl[r * L + j];
                    bels[v * L + j] = nb[r * L + j];
                }
                if (nbest[r] != best[v]) {
                    best[v] = nbest[r];
                    ++changed;
                }
            }
        }
        if ((double)changed <= tol * (double)n) break;
    }
    free(nl);
    free(nb);
    free(ns);
    free(nbest);
    scratch_free(&s);
    return it;
}

/* ---------------------------------------------------------------------- */
/* SLPA (slpa.py)                                                         */
/* ---------------------------------------------------------------------- */

/* slpa.py:51-66: most frequent, smallest id on frequency ties */
static int64_t modal_label(const int64_t* row, int64_t filled) {
    int64_t best = -1, best_c = 0;
    for (int64_t i = 0; i < filled; ++i) {
        int64_t lab = row[i], c = 0;
        for (int64_t j = 0; j < filled; ++j) c += row[j] == lab;
        if (c > best_c || (c == best_c && lab < best)) {
            best = lab;
            best_c = c;
        }
    }
    return best;
}

/* Counter RNG for the speaker draw (GPU rule): keyed by the round t, the
 * listener v and the speaker's index k among v's non-self arcs (scan
 * order); the slot is the hash mod filled[u]. */
uint32_t or_speak_hash(uint32_t seed, uint32_t t, uint32_t listener, uint32_t e) {
    return or_tie_hash(seed ^ 0x53504B52u, t, listener, e);
}

/*
 * SLPA with the batched schedule over index order (slpa.py:99 visits
 * v = 0..n-1; batches == n with tie OR_TIE_XORSHIFT / OR_TIE_SCAN_FIRST and
 * reference draws reproduces _slpa_seq).  With tie OR_TIE_XORSHIFT or
 * strict+xorshift speakers (speaker_rng = 0) draws follow the reference
 * stream; speaker_rng = 1 uses or_speak_hash (GPU rule).  slots n x T
 * row-major (slot 0 = own id), filled n, prev n, all in/out; labels n out
 * (projection, slpa.py:147-150).  Returns iterations.
 */
int or_slpa(int64_t n, const int64_t* off, const int64_t* nbr, const double* w, int64_t T,
            int64_t batches, int tie, int speaker_rng, uint32_t seed, double tol, int64_t* slots,
            int64_t* filled, int64_t* prev, int64_t* labels) {
    if (n == 0) return 0;
    if (batches <= 0 || batches > n) batches = n;
    int64_t bs = (n + batches - 1) / batches;
    scratch_t s;
    if (scratch_init(&s, n)) return -1;
    int64_t* fresh = (int64_t*)malloc((size_t)bs * sizeof(int64_t));
    if (!fresh) return -1;
    uint32_t xs = or_mix_seed(seed, 0);
    int it = 0;
    for (int64_t t = 1; t < T; ++t) {
        ++it;
        int64_t repeats = 0;
        for (int64_t b0 = 0; b0 < n; b0 += bs) {
            int64_t b1 = b0 + bs < n ? b0 + bs : n;
            for (int64_t v = b0; v < b1; ++v) {
                int64_t count = 0;
                uint32_t spk = 0; /* index of the speaker among v's non-self arcs */
                for (int64_t e = off[v]; e < off[v + 1]; ++e) {
                    int64_t u = nbr[e];
                    if (u == v) continue; /* slpa.py:75 */
                    uint32_t j = speaker_rng ? or_speak_hash(seed, (uint32_t)t, (uint32_t)v, spk++) % (uint32_t)filled[u]
                                             : or_draw(&xs, (uint32_t)filled[u]);
                    int64_t lab = slots[u * T + j];
                    if (s.tally[lab] == 0.0) s.touched[count++] = lab;
                    s.tally[lab] += w ? w[e] : 1.0;
                }
                int64_t lab;
                if (count == 0)
                    lab = modal_label(slots + v * T, filled[v]);
                else {
                    lab = pick_from_tally(s.touched, s.tally, count, tie, &xs, seed, (uint32_t)t, (uint32_t)v);
                    untally(&s, count);
                }
                fresh[v - b0] = lab;
            }
            for (int64_t v = b0; v < b1; ++v) {
                int64_t lab = fresh[v - b0];
                slots[v * T + filled[v]] = lab;
                filled[v] += 1;
                if (lab == prev[v]) ++repeats;
                prev[v] = lab;
            }
        }
        if (t >= 2 && (double)repeats >= (1.0 - tol) * (double)n) break; /* slpa.py:109-110 */
    }
    for (int64_t v = 0; v < n; ++v) labels[v] = modal_label(slots + v * T, filled[v]);
    free(fresh);
    scratch_free(&s);
    return it;
}

/* ---------------------------------------------------------------------- */
/* modularity (quality.py:10-42), double precision                        */
/* ---------------------------------------------------------------------- */
double or_modularity(int64_t n, const int64_t* off, const int64_t* nbr, const double* w, const int64_t* labels,
                     double total) {
    if (n == 0 || total <= 0) return 0.0;
    double* wc = (double*)calloc((size_t)n, sizeof(double));
    double* dc = (double*)calloc((size_t)n, sizeof(double));
    for (int64_t v = 0; v < n; ++v) {
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
            int64_t u = nbr[e];
            double we = w ? w[e] : 1.0;
            double f = (u == v) ? 2.0 : 1.0;
            dc[labels[v]] += we * f;
            if (labels[u] == labels[v]) wc[labels[v]] += we * f;
        }
    }
    double q = 0.0;
    for (int64_t c = 0; c < n; ++c) q += wc[c] / total - (dc[c] / total) * (dc[c] / total);
    free(wc);
    free(dc);
    return q;
}

/* ------------------------------------------------------------------------
 * Benchmark graphs, built without the product library (bench.py's reference
 * arm and the generator cross-checks in tests/test_oracle_graphs.py).  The
 * reference ships no R-MAT / planted / grid generator;
 * these restate the seeded recipes of DESIGN.md §5 independently of the
 * product's native builders, and the canonical CSR form of the reference's
 * preprocess(from_arcs(...)) (graph.py:58-84,254-306: symmetric, duplicate
 * pairs merged, generated self-loops dropped, one unit self-loop per vertex,
 * rows sorted by neighbour id).
 * ---------------------------------------------------------------------- */

static inline uint64_t or_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* R-MAT pair i: bit level l (high to low) draws a 53-bit uniform from
 * splitmix64(key ^ 64 i + l) and takes quadrant a | b | c | d. */
int or_gen_rmat_pairs(int32_t scale, int64_t edges, double a, double b, double c, uint64_t seed, int64_t* src,
                      int64_t* dst) {
    if (scale < 1 || scale > 30 || edges < 0) return -1;
    const double two53 = 9007199254740992.0;
    const uint64_t t1 = (uint64_t)(a * two53), t2 = (uint64_t)((a + b) * two53), t3 = (uint64_t)((a + b + c) * two53);
    const uint64_t key = or_splitmix64(seed ^ 0x524D4154ull);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < edges; ++i) {
        uint64_t row = 0, col = 0;
        for (int l = scale - 1; l >= 0; --l) {
            const uint64_t r = or_splitmix64((key ^ ((uint64_t)i << 6)) + (uint64_t)l) >> 11;
            /* quadrants: [0,a) top-left, [a,a+b) top-right, [a+b,a+b+c) bottom-left, rest bottom-right */
            const uint64_t down = r >= t2;
            const uint64_t right = (r >= t1 && r < t2) || r >= t3;
            row |= down << l;
            col |= right << l;
        }
        src[i] = (int64_t)row;
        dst[i] = (int64_t)col;
    }
    return 0;
}

/* LSD radix sort of 64-bit keys, 11-bit digits, skipping digits that are
 * constant over the input. */
static int radix_sort_u64(uint64_t* keys, int64_t count) {
    uint64_t* tmp = (uint64_t*)malloc((size_t)(count > 0 ? count : 1) * sizeof(uint64_t));
    if (!tmp) return -1;
    uint64_t *src = keys, *dst = tmp;
    for (int shift = 0; shift < 64; shift += 11) {
        int64_t hist[2048];
        memset(hist, 0, sizeof(hist));
        for (int64_t i = 0; i < count; ++i) ++hist[(src[i] >> shift) & 2047];
        int constant = 0;
        for (int d = 0; d < 2048; ++d)
            if (hist[d] == count) constant = 1;
        if (constant) continue;
        int64_t run = 0;
        for (int d = 0; d < 2048; ++d) {
            int64_t h = hist[d];
            hist[d] = run;
            run += h;
        }
        for (int64_t i = 0; i < count; ++i) dst[hist[(src[i] >> shift) & 2047]++] = src[i];
        uint64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != keys) memcpy(keys, src, (size_t)count * sizeof(uint64_t));
    free(tmp);
    return 0;
}

/* Canonical unit-weight CSR of an undirected pair list.  neighbors must
 * hold 2 * pairs + n entries; returns the arc count, or -1 on bad input /
 * allocation failure. */
int64_t or_csr_undirected(int64_t n, int64_t pairs, const int64_t* u, const int64_t* v, int64_t* offsets,
                          int64_t* neighbors) {
    if (n < 0 || n >= ((int64_t)1 << 31) || pairs < 0) return -1;
    uint64_t* keys = (uint64_t*)malloc((size_t)(pairs > 0 ? pairs : 1) * sizeof(uint64_t));
    if (!keys) return -1;
    int64_t k = 0;
    for (int64_t i = 0; i < pairs; ++i) {
        if (u[i] < 0 || v[i] < 0 || u[i] >= n || v[i] >= n) {
            free(keys);
            return -1;
        }
        if (u[i] == v[i]) continue; /* generated self-loops dropped */
        const uint64_t lo = (uint64_t)(u[i] < v[i] ? u[i] : v[i]), hi = (uint64_t)(u[i] < v[i] ? v[i] : u[i]);
        keys[k++] = (lo << 32) | hi;
    }
    if (radix_sort_u64(keys, k)) {
        free(keys);
        return -1;
    }
    int64_t uniq = 0;
    for (int64_t i = 0; i < k; ++i)
        if (uniq == 0 || keys[i] != keys[uniq - 1]) keys[uniq++] = keys[i];
    for (int64_t r = 0; r <= n; ++r) offsets[r] = 0;
    for (int64_t i = 0; i < uniq; ++i) {
        ++offsets[(keys[i] >> 32) + 1];
        ++offsets[(keys[i] & 0xFFFFFFFFull) + 1];
    }
    for (int64_t r = 0; r < n; ++r) offsets[r + 1] += offsets[r] + 1; /* + the self-loop */
    /* Row r holds its smaller neighbours, itself, then its larger ones.  In
     * (lo, hi) order the pairs with a given hi arrive by ascending lo and
     * those with a given lo by ascending hi, so three passes fill every row
     * in ascending neighbour order. */
    int64_t* fill = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!fill) {
        free(keys);
        return -1;
    }
    for (int64_t r = 0; r < n; ++r) fill[r] = offsets[r];
    for (int64_t i = 0; i < uniq; ++i) neighbors[fill[keys[i] & 0xFFFFFFFFull]++] = (int64_t)(keys[i] >> 32);
    for (int64_t r = 0; r < n; ++r) neighbors[fill[r]++] = r;
    for (int64_t i = 0; i < uniq; ++i) neighbors[fill[keys[i] >> 32]++] = (int64_t)(keys[i] & 0xFFFFFFFFull);
    free(fill);
    free(keys);
    return offsets[n];
}

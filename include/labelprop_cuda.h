/*
 * labelprop_cuda.h -- C-ABI of the B200 label-propagation engine
 * (liblabelprop_cuda.so, built from paper_2301_09125_b200/csrc).
 *
 * This is the drop-in boundary for the reference's hot path.  In the
 * reference (/root/reference/pkg/src/labelprop) the boundary is the numba
 * call site: rak_detect() hands raw numpy buffers to the compiled kernel
 *
 *     iterations = _rak_seq(offsets, neighbors, weights, labels, order,
 *                           strict, tolerance, max_iterations,
 *                           states, tally, touched)            (rak.py:177-181)
 *     iterations = _rak_par(..., tallies, touches, CHUNK)       (rak.py:188-192)
 *
 * and the kernel mutates `labels` in place and returns the sweep count.
 * lp_rak_run() replaces exactly that call: same CSR arrays (int64 offsets,
 * int64 neighbours, float64 weights -- the dtypes of graph.Graph,
 * graph.py:44-50), same order array (prng.shuffled_indices, rak.py:171),
 * same tolerance / max_iterations / strict semantics, labels written back
 * in place, iteration count returned.  The per-thread scratch (states,
 * tally, touched) disappears: the engine owns its device scratch.
 *
 * The CSR is uploaded once into an lp_graph handle (lp_graph_create) and
 * reused across runs, which is how a Python Graph object (immutable,
 * graph.py:34) maps onto device memory.
 *
 * COPRA (copra.py:124-176 / _copra_par :179-237) and SLPA (slpa.py:91-144)
 * follow the same pattern: lp_copra_run / lp_slpa_run.
 *
 * Conventions: plain C types only; host pointers unless a flag says
 * otherwise; return 0 on success, a negative LP_ERR_* code on failure with
 * a thread-local message in lp_last_error().  Python maps LP_ERR_INVALID to
 * ValueError and every other code to RuntimeError.  A
 * handle is not re-entrant (one stream per handle), matching the
 * reference's one-run-at-a-time contract.
 */
#ifndef LABELPROP_CUDA_H
#define LABELPROP_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LP_OK 0
#define LP_ERR_INVALID (-1)     /* bad argument            -> ValueError   */
#define LP_ERR_CUDA (-2)        /* CUDA failure / no GPU   -> RuntimeError */
#define LP_ERR_NOMEM (-3)       /* device allocation       -> RuntimeError */
#define LP_ERR_UNSUPPORTED (-4) /* e.g. >= 2^32 arcs       -> RuntimeError */

/* Tie rules (rak.py:57-84).  SCAN_FIRST is the reference's strict mode:
 * the first maximum-weight label in CSR scan order.  RANDOM is the
 * non-strict mode with a counter-based RNG (the reference's xorshift
 * stream order depends on a sequential visit and cannot be replayed by a
 * parallel sweep).  MIN_LABEL is the smallest label
 * among the maxima (BASELINE config-0 wording). */
#define LP_TIE_SCAN_FIRST 0
#define LP_TIE_RANDOM 1
#define LP_TIE_MIN_LABEL 2

/* Weight handling chosen at upload (lp_graph_info.weight_mode). */
#define LP_WEIGHTS_UNIT 0  /* all weights 1: integer counts               */
#define LP_WEIGHTS_FIXED 1 /* float32-exact weights: exact 64-bit sums   */
#define LP_WEIGHTS_FLOAT 2 /* anything else: float32 sums (approximate) */

typedef struct lp_graph lp_graph;

typedef struct lp_graph_info {
    int64_t vertex_count;
    int64_t edge_count;
    int32_t weight_mode;  /* LP_WEIGHTS_* */
    int32_t fixed_shift;  /* fixed-point scale 2^shift (FIXED mode)     */
    int64_t max_degree;
    int64_t device_bytes; /* device memory held by the handle            */
    int32_t device;
    int32_t reserved[7];
} lp_graph_info;

/* lp_rak_opts.flags */
#define LP_RAK_PROFILE 1 /* time every kernel launch with CUDA events (per-bin stats) */

typedef struct lp_rak_opts {
    double tolerance;       /* (0, 1]; stop when changed <= tolerance * n   */
    int32_t max_iterations; /* >= 1                                          */
    int32_t tie;            /* LP_TIE_*                                      */
    int64_t batches;        /* schedule: 0 or n = the reference's in-place
                               visit order (exact asynchronous semantics);
                               1 = synchronous sweep; B = B snapshot batches */
    uint32_t seed;          /* RakParams.seed: RNG key for LP_TIE_RANDOM     */
    int32_t flags;          /* LP_RAK_*                                      */
    int64_t reserved[6];
} lp_rak_opts;

/* SLPA (slpa.py SlpaParams :34-48).  Speaking rounds t = 1 .. T-1 over the
 * identity visit order (slpa.py:99), self-loops silent (:75). */
typedef struct lp_slpa_opts {
    double tolerance;       /* (0, 1]; stop once repeats >= (1-tol) * n, t >= 2 */
    int32_t memory_size;    /* T >= 2                                        */
    int32_t tie;            /* LP_TIE_SCAN_FIRST (strict) / LP_TIE_RANDOM     */
    int64_t batches;        /* 0 or n = the reference's in-place sweep; 1 = synchronous */
    uint32_t seed;          /* speaker draws and random ties (counter RNG)   */
    int32_t flags;          /* LP_RAK_PROFILE                                */
    int64_t reserved[6];
} lp_slpa_opts;

/* COPRA (copra.py CopraParams :34-50).  Sweeps over the identity visit
 * order (copra.py:134), self arcs skipped (:137-139). */
typedef struct lp_copra_opts {
    double tolerance;       /* (0, 1]; stop when best labels changed <= tolerance * n */
    int32_t max_labels;     /* k in 1 .. 32                                  */
    int32_t max_iterations; /* >= 1                                          */
    int64_t batches;        /* 0 or n = the reference's in-place sweep; 1 = synchronous */
    uint32_t seed;          /* fallback ties (counter RNG)                   */
    int32_t flags;          /* LP_RAK_PROFILE                                */
    int64_t reserved[6];
} lp_copra_opts;

/* Kernel slots of the engine, index of the lp_run_stats
 * bin_* arrays.  A vertex is routed each round by its degree d and its
 * estimated distinct neighbour labels. */
#define LP_BIN_HUB 0   /* 16-warp block per (vertex, label partition | arc slice) */
#define LP_BIN_TEAM 1  /* 8-warp block per vertex, est <= 2048, d <= 16384   */
#define LP_BIN_WARP 2  /* warp per vertex, est <= 256, d <= 2048              */
#define LP_BIN_SMALL 3 /* thread per vertex, d <= 16                          */

typedef struct lp_run_stats {
    int32_t iterations;     /* sweeps run (rak.py:94-95 semantics)          */
    int32_t rounds;         /* device rounds over all sweeps                */
    double kernel_ms;       /* device time of the sweep loop (CUDA events)  */
    double plan_ms;         /* device time spent (re)building the plan      */
    int64_t arcs_scanned;   /* arcs actually evaluated over all rounds      */
    int64_t arcs_dense;     /* edge_count * iterations (dense-equivalent)   */
    int32_t launches;       /* sweep kernels launched (excl. copies/memsets) */
    int32_t reserved0;
    double bin_ms[4];       /* LP_RAK_PROFILE: summed launch time per slot  */
    int64_t bin_launches[4];
    int64_t bin_arcs[4];    /* arcs scanned per bin                         */
    int64_t bin_vertices[4];/* vertex evaluations per bin                   */
    double aux_ms;          /* LP_RAK_PROFILE: routing kernels' time        */
    double gather_ms;       /* LP_RAK_PROFILE: phase-1 label gather time    */
    int64_t arcs_gathered;  /* arcs whose neighbour label phase 1 gathered  */
    int64_t gather_launches;
    int64_t flags;          /* LP_STATS_FUSED: the tally kernels gathered the
                               neighbour labels themselves (no phase 1)    */
} lp_run_stats;
#define LP_STATS_FUSED 1

/* Upload a CSR graph.  offsets[n+1], neighbors[m] (int64, rows sorted by
 * neighbour id -- graph.py:39-41), weights[m] float64 or NULL (= all 1).
 * device < 0 selects the calling thread's current CUDA device. */
int lp_graph_create(int64_t n, int64_t m, const int64_t* offsets, const int64_t* neighbors,
                    const double* weights, int32_t device, lp_graph** out);
int lp_graph_destroy(lp_graph* g);
int lp_graph_get_info(const lp_graph* g, lp_graph_info* info);
/* The handle's CUDA stream (cudaStream_t), for callers that time or order
 * work against it. */
void* lp_graph_stream(lp_graph* g);

/* RAK.  order[n]: visit permutation (host int64, prng.shuffled_indices);
 * NULL means shuffled_indices(n, opts->seed) computed by the library.
 * labels[n]: in = initial labels (NULL-safe: pass labels_init = NULL for
 * arange(n), rak.py:168), out = final labels (host int64).
 * changed_per_iter: NULL or max_iterations entries.  stats: NULL or out. */
int lp_rak_run(lp_graph* g, const lp_rak_opts* opts, const int64_t* order, const int64_t* labels_init,
               int64_t* labels_out, int64_t* changed_per_iter, lp_run_stats* stats);

/* Same sweep, labels kept on the device (no host transfers; for timing
 * with inputs resident in HBM).  lp_labels_download() copies them out. */
int lp_rak_run_resident(lp_graph* g, const lp_rak_opts* opts, const int64_t* order, lp_run_stats* stats);
int lp_labels_download(lp_graph* g, int64_t* labels_out);

/* SLPA: replaces _slpa_seq/_slpa_par + _project (slpa.py:91-150).
 * labels_out[n]: modal label of every memory (NULL: skip); slots_out[n*T]:
 * the memories, row-major, unfilled slots 0 (NULL: skip); every memory
 * holds stats->iterations + 1 labels.  repeats_per_iter: NULL or T-1. */
int lp_slpa_run(lp_graph* g, const lp_slpa_opts* opts, int64_t* labels_out, int64_t* slots_out,
                int64_t* repeats_per_iter, lp_run_stats* stats);

/* COPRA: replaces _copra_seq/_copra_par (copra.py:124-237).  best_out[n]
 * (required): the best label per vertex (the disjoint projection);
 * labs_out[n*k] / bels_out[n*k] (both or neither): label sets sorted by
 * label, belongings float64, entries past sizes_out[v] zero; sizes_out[n]
 * optional.  changed_per_iter: NULL or max_iterations entries.  Belongings
 * use float64 arithmetic in the reference's order (bit-exact to the CPU
 * restatement of the same schedule). */
int lp_copra_run(lp_graph* g, const lp_copra_opts* opts, int64_t* labs_out, double* bels_out, int64_t* sizes_out,
                 int64_t* best_out, int64_t* changed_per_iter, lp_run_stats* stats);

/* Modularity (quality.py:10-42) on the device, float64 accumulators:
 * labels[n] host int64, or NULL for the labels of the last RAK run on this
 * handle; total_weight = Graph.total_weight.  Equals the reference's value
 * up to float64 summation order (exactly, for integer weights, up to the
 * final sum of squares). */
int lp_modularity(lp_graph* g, const int64_t* labels, double total_weight, double* q_out);

/* Calibration (device time per pass, ms): mode 0 streams the neighbour
 * indices of the active rows once; mode 1 also gathers every neighbour's
 * label (the sweep's memory traffic without the tally).  Needs a plan
 * (run a detection first). */
int lp_calibrate(lp_graph* g, int32_t mode, int32_t reps, double* ms_out);

/* Host utilities (no GPU needed).  lp_shuffled_indices reproduces the
 * reference's prng.shuffled_indices (prng.py:82-94) byte for byte. */
int lp_shuffled_indices(int64_t n, uint32_t seed, int64_t* out);
/* Native graph builders for the benchmark inputs (host, OpenMP).
 * lp_gen_rmat: `edges` R-MAT pairs on 2^scale vertices, quadrant
 * probabilities a, b, c (d = 1-a-b-c), counter-based RNG keyed by seed.
 * lp_csr_build_undirected: canonical preprocessed CSR (what
 * preprocess(from_arcs(...)) returns for unit weights, graph.py:254-306)
 * from an undirected pair list; neighbors must hold 2*pairs + n entries,
 * *m_out receives the arc count. */
int lp_gen_rmat(int32_t scale, int64_t edges, double a, double b, double c, uint64_t seed, int64_t* src,
                int64_t* dst);
int lp_csr_build_undirected(int64_t n, int64_t pairs, const int64_t* u, const int64_t* v, int64_t* offsets,
                            int64_t* neighbors, int64_t* m_out);
/* The same builders on the GPU (identical arrays):
 * lp_gen_rmat_csr generates the R-MAT pairs of lp_gen_rmat on the device
 * and builds the canonical CSR; lp_csr_build_undirected_gpu builds it from a
 * host pair list.  neighbors_cap = capacity of neighbors (2*pairs + n
 * suffices); device < 0 = the calling thread's current device. */
int lp_gen_rmat_csr(int32_t scale, int64_t edges, double a, double b, double c, uint64_t seed, int32_t device,
                    int64_t* offsets, int64_t* neighbors, int64_t neighbors_cap, int64_t* m_out);
int lp_csr_build_undirected_gpu(int64_t n, int64_t pairs, const int64_t* u, const int64_t* v, int32_t device,
                                int64_t* offsets, int64_t* neighbors, int64_t neighbors_cap, int64_t* m_out);
/* Page-lock a host range for fast uploads / downloads (cudaHostRegister). */
int lp_host_register(void* ptr, int64_t bytes);
int lp_host_unregister(void* ptr);
const char* lp_last_error(void);
const char* lp_version(void);
int lp_device_count(int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* LABELPROP_CUDA_H */

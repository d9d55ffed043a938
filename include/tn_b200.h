/*
 * tn_b200.h -- C ABI of the B200-native sliced bucket-elimination contractor
 * for QAOA MaxCut tensor networks (arXiv:2012.02430, "Tensor Network Quantum
 * Simulator With Step-Dependent Parallelization").
 *
 * Citations are PAPER.md line numbers (+ section / equation) of the paper text
 * in the reference bundle.  The library is libtnb200.so; every entry point is
 * extern "C", takes plain pointers and sizes, never throws, and returns a
 * tn_status (0 = OK, < 0 = error; tn_last_error() has a thread-local message).
 *
 * Memory ownership: the caller owns every buffer passed in (host arrays,
 * device workspace, result arrays) and the CUDA stream.  A tn_plan owns its
 * host tables and, lazily, one small device copy of its step tables per
 * device (freed by tn_plan_free).  The library never calls cudaMalloc for
 * tensors: all intermediates live in the caller's workspace (`ws`).
 * "Device" pointers below are CUDA global-memory pointers on the current
 * device; "host" pointers are ordinary CPU memory.
 */
#ifndef TN_B200_H
#define TN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tn_plan tn_plan; /* opaque, immutable after load, shareable across threads */

typedef enum { TN_C64 = 0, TN_C128 = 1 } tn_dtype; /* complex64 / complex128 storage + arithmetic */

typedef enum {
  TN_OK = 0,
  TN_E_INVAL = -1,    /* bad argument: p mismatch, begin > end, short workspace, null pointer */
  TN_E_PLAN = -2,     /* malformed / version-mismatched plan, order misses a live label,
                         n exceeds the live vertex count */
  TN_E_TOO_WIDE = -3, /* contraction width above opts->max_width or device memory */
  TN_E_NOMEM = -4,    /* host allocation failed */
  TN_E_CUDA = -5,     /* a CUDA runtime call or kernel launch failed (message has the CUDA error) */
  TN_E_DTYPE = -6     /* unsupported dtype */
} tn_status;

typedef enum { TN_KIND_AMPLITUDE = 0, TN_KIND_ENERGY = 1 } tn_kind;
typedef enum {
  TN_ORDER_MIN_FILL = 0,    /* greedy, fewest fill-in edges first */
  TN_ORDER_MIN_DEGREE = 1,  /* greedy, lowest degree first */
  TN_ORDER_RGREEDY = 2,     /* "rgreedy": p(v) ~ exp(-N_G(v)/tau), best of q runs */
  TN_ORDER_RGREEDY_FILL = 3 /* the same Boltzmann sampling on the fill-in count (extension) */
} tn_orderer;

/* Planner options (§5.1 ordering; §5.3 step-dependent slicing). */
typedef struct {
  int32_t kind;           /* tn_kind */
  int32_t orderer;        /* tn_orderer: greedy min-fill, or min-degree ("contracts the lowest-degree
                             vertex"). Ties: min-fill -> lower degree -> smaller label;
                             min-degree -> smaller label. */
  int32_t n_sliced;       /* n of §5.3: number of sliced indices (0 = no slicing). Amplitude only. */
  int32_t r;              /* r of §5.3: indices sliced per round (r == n: one slice step s; the
                             paper's 210-qubit run). 0 means r = n. */
  int32_t max_width;      /* > 0: fail with TN_E_TOO_WIDE if the contraction width exceeds it */
  int32_t small_log2;     /* steps whose output has <= small_log2 indices run in the batched
                             interpreter kernel; < 0 selects the default (12) */
  int32_t rg_q;           /* rgreedy: number of randomized runs q (>= 1; 0 -> 8); the deterministic
                             greedy run is always included, so the result is never worse */
  int32_t rg_tau_milli;   /* rgreedy: temperature tau x 1000 (0 -> tau = 0.5) */
  uint32_t rg_seed;       /* rgreedy: seed (runs are deterministic for a seed) */
  int32_t n_open;         /* a: output wires left open (amplitude plans, §6): the
                             result is the batch of 2^a amplitudes <x 0_rest|U|0^N>, bit b of the
                             batch index x = output bit of the b-th open qubit (ascending).  The open
                             indices form a clique in the line graph and are never eliminated or
                             sliced.  0 <= a <= 20; 0 = single amplitude */
  const int32_t* open_qubits; /* host int32[n_open]: distinct qubits in [0, n_qubits) (any order) */
} tn_build_opts;

typedef struct {
  int32_t kind, n_qubits, p, n_edges;
  int32_t width;          /* contraction width c = max_i N_{G_i}(v_i) over executed steps */
  int32_t unsliced_width; /* width of the planner's full greedy order before slicing */
  int32_t k;              /* number of sliced indices; 2^k slices (Eq. 1) */
  int32_t slice_step;     /* s: length of the shared, unsliced prefix */
  int32_t n_programs;     /* 1 (amplitude) or E = #edges (energy: one light cone per edge) */
  int32_t n_labels;       /* live indices of the (first) network */
  uint64_t n_slices;      /* 2^k */
  uint64_t prefix_steps;  /* bucket steps run once per call (before slicing) */
  uint64_t steps_per_slice;
  uint64_t launches_prefix;    /* kernel launches of the prefix */
  uint64_t launches_per_slice; /* kernel launches per slice (incl. the per-slice finalize) */
  size_t workspace_bytes[2];   /* per tn_dtype: bytes of device workspace needed by every call */
  double pred_bytes_per_slice[2]; /* algorithmic bytes of one slice: sum over launches of
                                     (inputs read once + output written once) x sizeof(dtype); a
                                     fused group counts its inputs and final output, a producer ->
                                     consumer pair (OP_GROUP_FEED) not the intermediate it never
                                     writes (tn_plan_steps gives the per-step, unfused bytes) */
  double pred_bytes_prefix[2];
  double pred_bytes_big_per_slice[2]; /* the part of pred_bytes_per_slice in standalone launches */
  uint64_t big_launches_per_slice;    /* standalone bucket-kernel launches per slice */
  int32_t slices_batchable;  /* 1: every per-slice step runs in the interpreter, so slices run
                                batched (one CTA per slice) when the workspace holds windows */
  int32_t n_open;            /* a: results are batches of 2^a amplitudes (tn_build_opts.n_open) */
} tn_plan_info_t;

/* ---------------------------------------------------------------- planning (host only) */
/* Build a plan for the QAOA MaxCut instance (graph, depth p).  edges: host int32[2*n_edges]
 * (pairs i<j or j<i, 0-based).  kind AMPLITUDE: the single amplitude sigma = <0^N|U|0^N>
 * (§5) as ONE network with live indices w(q,l) = l*N+q, l < p;
 * kind ENERGY: one reverse-light-cone <Z_u Z_v> network per edge.
 * Output: *buf (host, library-allocated; release with tn_buffer_free), *len bytes.
 * The plan does not depend on (gamma, beta): it is reused across parameters. */
tn_status tn_plan_build(int32_t n_qubits, int32_t n_edges, const int32_t* edges, int32_t p,
                        const tn_build_opts* opts, void** buf, size_t* len);
void tn_buffer_free(void* buf);

/* Step-dependent slicing scan (Fig. slice_algo): for the FIRST slicing round of
 * the amplitude network of (graph, p) with opts->n_sliced = n indices (rounds of opts->r), every
 * candidate slice step s in [0, peak] (reading A8) with the contraction width and the predicted
 * cost sum_i 2^{degree_i} (prefix once + 2^n x residual) of the plan that slices at s -- the data
 * of the paper's Fig. hist_of_cost ("difference ... goes up to 9").  Host only.
 * opts: as tn_plan_build (kind must be AMPLITUDE, 1 <= n_sliced <= 30).  Outputs: host arrays
 * s_out / width_out (int32[cap]) and cost_out (double[cap]) receive the first min(cap, count)
 * candidates in ascending s; *n_out = count; *peak_out (may be NULL) = the peak step of the
 * unsliced order.  cap = 0 queries the count.  Errors: TN_E_INVAL (bad argument), TN_E_PLAN
 * (n exceeds the live vertex count). */
tn_status tn_slice_scan(int32_t n_qubits, int32_t n_edges, const int32_t* edges, int32_t p,
                        const tn_build_opts* opts, int32_t* s_out, int32_t* width_out,
                        double* cost_out, int32_t cap, int32_t* n_out, int32_t* peak_out);

/* Parse + validate a plan buffer (host; the contract input of SPEC.md:290-298: a network plus an
 * elimination order that covers every live label -- "order misses a live label", is
 * raised by tn_plan_build).  Checks magic / version, record counts against the buffer length,
 * every step's output and input ranges against the arena, and the op / scalar / program records.
 * Caller owns *out; free with tn_plan_free.
 * Errors: TN_E_INVAL (null argument), TN_E_PLAN (malformed or version-mismatched buffer). */
tn_status tn_plan_load(const void* buf, size_t len, tn_plan** out);
void tn_plan_free(tn_plan* plan);
tn_status tn_plan_info(const tn_plan* plan, tn_plan_info_t* out);

/* The schedule as data (amplitude plans): host arrays sized by tn_plan_info:
 * prefix[slice_step] labels, sliced[k] labels (ascending: bit b of slice id j is the value of
 * sliced[b], reading A13), residual[n_labels - n_open - slice_step - k] labels,
 * degrees[n_labels - n_open - k]
 * (N_{G_i}(v_i) of the executed steps).  Any pointer may be NULL. */
tn_status tn_plan_schedule(const tn_plan* plan, int32_t* prefix, int32_t* sliced, int32_t* residual,
                           int32_t* degrees);

/* Per-step description of the lowered bucket program (Fig. contract_cost: the
 * cost of every elimination step).  out: host array of cap records; *n = number of steps. */
typedef struct {
  int32_t phase;          /* 0: shared prefix (run once), 1: per slice */
  int32_t label;          /* eliminated index */
  int32_t out_rank;       /* bits of the output in this phase */
  int32_t degree;         /* N_{G_i}(v_i): indices of the output incl. sliced ones in phase 0 */
  int32_t n_in;
  int32_t inplace;        /* output aliases the first input's lower half */
  int32_t standalone;     /* 1: own k_bucket launch; 2: part of a fused reduce chain (k_chain);
                             3: part of a fused merge group (k_group_t); 0: inside an interpreter run */
  int32_t in_rank[8];     /* bits of each input read per slice */
  uint64_t in_out_mask[8];
  int32_t in_pv[8];
  double bytes_c64;       /* algorithmic bytes (inputs + output) at complex64 */
} tn_step_info_t;
tn_status tn_plan_steps(const tn_plan* plan, tn_step_info_t* out, int64_t cap, int64_t* n);

/* ---------------------------------------------------------------- contraction (device) */
/* The amplitude sigma = <0^N|U(gamma, beta)|0^N> of the QAOA circuit U (§5: "the
 * tensor expression ... with boundary indices fixed"; sliced plans: all 2^k slices of Eq. (1),
 * PAPER.md:519-524, summed locally).  gamma, beta: host double[p].
 * ws: device buffer of >= workspace_bytes[dtype] bytes (e.g. torch.empty).  stream: cudaStream_t
 * (NULL = legacy default stream).  out: host double[2 * 2^a] = {Re, Im} of batch entry x at
 * out[2x], out[2x+1] (a = n_open; a = 0: the single amplitude sigma), 2^{-N/2} applied in FP64
 * (reading A15).  Synchronous with respect to `stream` on return. */
tn_status tn_contract(const tn_plan* plan, tn_dtype dtype, const double* gamma, const double* beta,
                      int32_t p, void* ws, size_t ws_bytes, void* stream, double* out);

/* Slices [begin, end) of a sliced plan, Eq. (1): runs the shared prefix once,
 * then every slice; writes the complex128 result of slice j, batch entry x (x < 2^a, a = n_open)
 * into device double partials_dev[2(j 2^a + x)], partials_dev[2(j 2^a + x) + 1] (2^{-N/2}
 * applied) and leaves other entries untouched.
 * Asynchronous on `stream`.  The caller zero-fills, all-reduces (torch.distributed / NCCL) and
 * sums with tn_sum_partials.  When ws_bytes holds L >= 2 windows of per-slice tensors
 * (tn_workspace_bytes(plan, dtype, L)), slice j of the range runs on lane (j - begin) mod L:
 * lane 0 on `stream`, lane l >= 1 on a library-owned stream in window l, all forked from and
 * joined back into `stream` (results identical to one lane).  Lanes = min(L, TNB_LANES
 * environment variable, default 16; TNB_ONE_LANE=1 forces one). */
tn_status tn_contract_sliced(const tn_plan* plan, tn_dtype dtype, const double* gamma,
                             const double* beta, int32_t p, uint64_t begin, uint64_t end, void* ws,
                             size_t ws_bytes, void* stream, double* partials_dev);

/* Fixed-order pairwise sum over j of the per-slice results (host; bit-identical for any partition
 * of the slices across GPUs), per batch entry x: partials_host as written by
 * tn_contract_sliced (double[2 n_slices 2^a]); out: host double[2 * 2^a]. */
tn_status tn_sum_partials(const tn_plan* plan, const double* partials_host, double* out);

/* QAOA MaxCut energy <psi|C|psi> as the sum of per-edge <Z_u Z_v> (§3.2: each
 * term evaluated on its own reverse-light-cone network).  Energy plan: all E light-cone networks
 * contracted in ONE batched launch.  zz: host double[E]
 * (Re <Z_u Z_v> per edge in the graph's edge order), zz_imag_max: host double (max |Im|, ~0),
 * energy: host double = sum_e (1 - zz[e]) / 2 (reading A3).  Synchronous on return. */
tn_status tn_energy(const tn_plan* plan, tn_dtype dtype, const double* gamma, const double* beta,
                    int32_t p, void* ws, size_t ws_bytes, void* stream, double* zz,
                    double* zz_imag_max, double* energy);

/* Parameter-batched energy (the QAOA outer loop reuses one plan across parameters,
 * PAPER.md:671-673): `batch` sets of angles, gammas/betas host double[batch * p] (set b at
 * [b*p, b*p + p)), all E x batch light cones in ONE launch.  ws >= tn_workspace_bytes(plan, dtype,
 * batch).  zz: host double[batch * E]; zz_imag_max, energy: host double[batch] (may be NULL). */
tn_status tn_energy_batch(const tn_plan* plan, tn_dtype dtype, const double* gammas,
                          const double* betas, int32_t p, uint64_t batch, void* ws, size_t ws_bytes,
                          void* stream, double* zz, double* zz_imag_max, double* energy);

/* Workspace bytes for `batch` windows: energy plans -- `batch` parameter sets (tn_energy_batch);
 * amplitude plans whose per-slice steps all run in the interpreter -- up to `batch` slices per
 * launch in tn_contract_sliced / tn_contract (slice batching; the library uses as
 * many windows as the given ws_bytes holds); other amplitude plans -- two slice lanes when
 * batch >= 2 (see tn_contract_sliced).  batch <= 1 gives workspace_bytes[dtype]. 0 on error. */
size_t tn_workspace_bytes(const tn_plan* plan, tn_dtype dtype, uint64_t batch);

/* One bucket step -- "elimination of vertex (index) v" (§4.2) -- on caller
 * tensors:  out[o] = sum_{x in {0,1}} prod_t in_t[ins(pext(o, out_mask[t]), pv[t], x)],
 * where pext gathers the output bits selected by out_mask[t] (in order) and ins inserts the summed
 * bit x at bit position pv[t] of input t.  Input t has popcount(out_mask[t]) + 1 bits.
 * in_dev: host array of n_in device pointers; out_dev: device pointer of 2^out_rank elements.
 * 1 <= n_in <= 8, 0 <= out_rank <= 40.  Asynchronous on `stream`. */
tn_status tn_eliminate(tn_dtype dtype, int32_t n_in, const void* const* in_dev,
                       const uint64_t* out_mask, const int32_t* pv, void* out_dev, int32_t out_rank,
                       void* stream);

/* A fused group: M consecutive bucket steps eliminating indices x_0 .. x_{M-1} in one pass --
 * the exact re-association of the same sum (PAPER.md:361-368 applied M times):
 *     out[o] = sum_{x in {0,1}^M} prod_t in_t[pext(o, out_mask[t]) + X_t(x)].
 * Input t holds the output bits out_mask[t] as its LOW bits (in order) and the summed indices
 * selected by x_mask[t] (bit i = x_i) as its TOP bits, x_0 the most significant (the plan's
 * elimination-order layout).  Input t has popcount(out_mask[t]) + popcount(x_mask[t]) bits;
 * every input must hold at least one summed index.  1 <= M <= 5, 1 <= n_in <= 8,
 * 11 <= out_rank <= 40.  kernel: 0 = the library's choice (as in a plan), 1 = k_gemm
 * (register-blocked batched complex GEMM on the FP32 pipes, c64 only), 2 = k_pair, 3 = k_group_t,
 * 4 = k_gemm_tc (the same GEMM on the tensor cores: tcgen05.mma kind::tf32 with a 3xTF32 split,
 * accumulators in TMEM; c64 only; needs >= 7 output bits held by one operand only, >= 3 by the
 * other only, 2 <= ... <= 32 summed values per tile row fitting shared memory), 5 = k_gemm_hm (the
 * same GEMM on the warp-level tensor cores: mma.sync m16n8k8 tf32 with a 3xTF32 split; c64 only;
 * needs M >= 2, out_rank >= 14, >= 4 output bits held by one operand only and >= 2 by the other
 * only, output bits 0 and 1 held by an operand, inputs other than the two holding no output bit);
 * TN_E_INVAL when the requested kernel does not take this shape.  Asynchronous on `stream`. */
tn_status tn_eliminate_group(tn_dtype dtype, int32_t M, int32_t n_in, const void* const* in_dev,
                             const uint64_t* out_mask, const uint32_t* x_mask, void* out_dev,
                             int32_t out_rank, int32_t kernel, void* stream);

/* Per-step device timing for the next calls on this plan (CUDA events on the launching stream).
 * enable != 0 turns it on.  tn_profile_read returns, for standalone bucket-kernel launches since
 * the last read: count, total milliseconds and total algorithmic bytes (host outputs). */
tn_status tn_profile_enable(tn_plan* plan, int32_t enable);
tn_status tn_profile_read(tn_plan* plan, uint64_t* launches, double* total_ms, double* total_bytes,
                          uint64_t* all_launches);

/* The per-launch records behind tn_profile_read (call it BEFORE tn_profile_read, which clears
 * them): one record per standalone launch with its plan step range, op kind (1 = single bucket
 * step, 2 = fused reduce chain, 3 = fused merge group, 4 = run of small steps in one CTA), the
 * kernel that ran it (1 = k_bucket, 2 = k_chain, 3 = k_group_t, 4 = k_pair, 5 = k_gemm,
 * 6 = k_chain_split, 7 = k_program, 8 = k_gemm_tc, 9 = k_gemm_fc: a producer group computed inside
 * its consumer's launch, whose record spans both groups' steps, 10 = k_fc_tc, 11 = k_gemm_hm),
 * device milliseconds,
 * algorithmic bytes (inputs read once + output written once) and flops (8 x 2^(out_rank + M): one
 * complex multiply-add per output element and summed value).  out: host array of cap records
 * (may be NULL to query *n). */
typedef struct {
  int32_t step_begin, step_end, kind, out_rank;
  double ms, bytes;
  int32_t kernel, pad;
  double flops;
} tn_prof_record_t;
tn_status tn_profile_records(tn_plan* plan, tn_prof_record_t* out, int64_t cap, int64_t* n);

const char* tn_last_error(void);
int32_t tn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TN_B200_H */

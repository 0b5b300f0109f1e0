/* latsum_b200 — C ABI of the B200-native lattice-sum hot path.
 *
 * Drop-in boundary for the reference's header-only C++ interface
 * (/root/reference/proj/include/latsum).  Each entry point cites the reference
 * function it replaces.  Conventions:
 *   - plain pointers and sizes, no C++ or torch types;
 *   - FP64, column-major, first index fastest, 0-based indices, int64 sizes;
 *   - every call returns int status (LATSUM_OK = 0) and never throws; the message
 *     of the last failure is latsum_last_error(ctx);
 *   - host pointers unless the name says _device; the context owns all device
 *     memory behind the opaque handles; one context per host thread.
 * There is no CPU fallback: every compute entry point runs CUDA kernels on the
 * context's device and fails with LATSUM_ERR_CUDA when no device is present.
 */
#ifndef LATSUM_B200_H
#define LATSUM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  LATSUM_OK = 0,
  LATSUM_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  LATSUM_ERR_WINDOW_OVERFLOW = 2,  /* WindowOverflowError (grid.hpp:87-98); mode in message */
  LATSUM_ERR_CUDA = 3,
  LATSUM_ERR_CUSOLVER = 4,
  LATSUM_ERR_OUT_OF_MEMORY = 5,
  LATSUM_ERR_LENGTH = 6,           /* std::length_error: dense guard (tensor3.hpp:101-105) */
  LATSUM_ERR_NOT_IMPLEMENTED = 7,  /* NotImplementedError (quadrature.hpp:110-112) */
  LATSUM_ERR_NCCL = 8,
  LATSUM_ERR_IO = 9                /* TensorIoError (tensor_io.hpp:27-29) */
};

enum { LATSUM_NEWTON = 0, LATSUM_YUKAWA = 1 }; /* kernel.hpp:17 KernelFamily (gauss type) */

enum { LATSUM_DEFLATE_NEVER = 0, LATSUM_DEFLATE_ALWAYS = 1, LATSUM_DEFLATE_AUTO = 2 };

/* latsum_rhosvd_ex flags: skip the dense core (r1 r2 r3 doubles; 518 GB for BASELINE
 * cfg5) and keep the projected factors P_l = Z_l^T A_l instead; entries and boxes are
 * then evaluated in projected-CP form, which equals the Tucker tensor. */
enum { LATSUM_RHOSVD_FACTORS_ONLY = 1, LATSUM_RHOSVD_CORE_SLABS = 2 };
/* LATSUM_RHOSVD_CORE_SLABS (row-sharded contexts): each rank forms and keeps only
 * rows [r1 q / P, r1 (q+1) / P) of mode 1 of the core, over the whole contraction, instead of
 * an all-reduced full core (BASELINE cfg5: 518 GB over 4-8 GPUs); entries and boxes add the
 * ranks' partial values with an all-reduce (every rank gets the full values);
 * latsum_tucker_core_slab returns the local slab, latsum_tucker_core refuses a slab. */

typedef struct latsum_ctx latsum_ctx;
typedef struct latsum_reference latsum_reference;
typedef struct latsum_canonical latsum_canonical;
typedef struct latsum_tucker latsum_tucker;

/* SpectralReport (rank_reduction.hpp:49-67) plus GPU-side diagnostics. */
typedef struct {
  int64_t chosen_ranks[3];
  double bound_abs, bound_rel, weight_norm, input_norm, stability_constant;
  int stability_ok;
  int tie_at_cutoff[3];
  int64_t n_singular[3];   /* length of singular_values[l] = min(N_l, M_c) */
  double cutoff_margin[3]; /* min(target - tail(r), tail(r-1) - target) / target; tolerance mode */
  int deflated[3];         /* 1 when the second (deflated) Gram pass ran for mode l */
  int gram_rows[3];        /* 1: Gram A A^T (N x N); 0: Gram A^T A over merged columns */
  int64_t gram_size[3];
  double ms_gram, ms_syevd, ms_deflate, ms_project, ms_core, ms_norm, ms_total; /* CUDA events */
  int64_t deflate_k1[3];   /* pass-1 directions kept (lambda > 1e-10 lambda_max) when deflated */
} latsum_spectral_report;

/* ------------------------------------------------------------------ context */
int latsum_ctx_create(int device, latsum_ctx** out);
void latsum_ctx_destroy(latsum_ctx* ctx);
const char* latsum_last_error(const latsum_ctx* ctx);
/* Run subsequent work on this cudaStream_t (NULL = the context's own stream). */
int latsum_ctx_set_stream(latsum_ctx* ctx, void* cuda_stream);
/* Return unused memory of the device's stream-ordered pool to the system, keeping at most
 * keep_bytes reserved (the context pre-grows the pool at creation and never releases it). */
int latsum_ctx_trim_pool(latsum_ctx* ctx, int64_t keep_bytes);
/* Host sink for the Tucker result of the following RHOSVDs on this context (cmd_sum writes
 * the result out, so its device->host copy belongs to the pipeline): the factors are copied
 * as soon as the bases exist and the core chunk by chunk right behind its contraction, on a
 * copy stream, so the transfer overlaps the core GEMMs.  core / factors[l] are host buffers
 * (pinned, cudaHostAlloc, for the overlap) of core_cap / factor_cap[l] doubles; a result
 * that does not fit stays on the device only.  core = NULL clears the sink.
 * latsum_tucker_sink_written tells whether a result was streamed (1) or not (0).           */
int latsum_ctx_set_host_sink(latsum_ctx* ctx, double* core, int64_t core_cap, double* const factors[3],
                             const int64_t factor_cap[3]);
int latsum_tucker_sink_written(const latsum_tucker* t);
int latsum_ctx_synchronize(latsum_ctx* ctx);
/* Number of kernels this context launched so far (its own kernels, not library ones). */
int64_t latsum_ctx_kernel_launches(const latsum_ctx* ctx);
/* In-house eigensolves redone with cuSOLVER syevd because their vectors failed the
 * orthogonality / finiteness check (this context and its workers, since creation). */
int64_t latsum_ctx_eig_fallbacks(const latsum_ctx* ctx);
/* Multi-GPU (one process per GPU): rank 0 creates an NCCL unique id, the caller
 * broadcasts it (e.g. torch.distributed), every rank calls latsum_ctx_init_comm.  The
 * context then runs latsum_rhosvd row-sharded over the grid index: each rank owns
 * N/nranks rows of every side matrix; Grams, U^T U, U^T A, P_l = Z_l^T A_l and the core
 * are all-reduced over NVLink, eigensolves run redundantly, Z is all-gathered.  NCCL is
 * bound at run time (dlopen libnccl.so.2). */
int latsum_comm_unique_id(unsigned char id[128]);
int latsum_ctx_init_comm(latsum_ctx* ctx, const unsigned char id[128], int rank, int nranks);
/* The same row-sharded reduction over caller-supplied host collectives instead of NCCL
 * (tests without a multi-GPU box: gloo ranks, or several contexts on one device driven from
 * host threads).  ar: in-place sum all-reduce of count doubles; ag: recv (nranks x count,
 * rank order) = all-gather of send.  channel identifies the calling stream: 0 = the
 * context, 1..4 = its four worker streams (the three modes and norm_f), which call
 * concurrently; a rank's calls on one channel come in the same order as every other rank's.
 * Callbacks return 0 on success.                                                       */
typedef int (*latsum_host_allreduce_fn)(void* user, int channel, double* buf, int64_t count);
typedef int (*latsum_host_allgather_fn)(void* user, int channel, const double* send, double* recv,
                                        int64_t count);
int latsum_ctx_init_host_comm(latsum_ctx* ctx, int rank, int nranks, latsum_host_allreduce_fn ar,
                              latsum_host_allgather_fn ag, void* user);
int latsum_ctx_comm_info(const latsum_ctx* ctx, int* rank, int* nranks);
/* Per-kernel-class CUDA-event timing: when on, every launch group is bracketed by
 * events on the context stream.  latsum_ctx_profile writes lines
 * "<tag> <launches> <total ms> <algorithmic work>" (FLOPs for gemm_*, bytes otherwise)
 * into buf and returns the full text length (call with buf=NULL to size it). */
int latsum_ctx_set_profiling(latsum_ctx* ctx, int on);
int64_t latsum_ctx_profile(latsum_ctx* ctx, char* buf, int64_t cap);

/* ------------------------------------------------------------------ host rules (no GPU)
 * quadrature.hpp:124-187 build_quadrature (gauss branch); nodes/weights hold 2M+1 values. */
int latsum_build_quadrature(int family, double lambda, int M, double step_constant,
                            double shell_a, double shell_A, double* nodes, double* weights);
/* quadrature.hpp:238-269 default_step_constant (53-point sweep, npts probe radii). */
double latsum_default_step_constant(int family, double lambda, int M, double shell_a,
                                    double shell_A, int npts);
/* reference.hpp:84-93 reference_shell of the doubled grid of (N, box). */
void latsum_reference_shell(const int64_t N[3], const double box[3], double shell[2]);
/* commands.cpp:254-260: the seeded probe stream of cmd_verify (std::mt19937_64(seed), one
 * uniform_int_distribution<Index>(0, dims[l] - 1) per mode, i, j, k per probe) -> probes n x 3,
 * so that a verification here visits the points `latsum verify` visits for the same seed. */
void latsum_verify_probes(uint64_t seed, const int64_t dims[3], int64_t n, int64_t* probes);

/* ------------------------------------------------------------------ stage 1
 * reference.hpp:95-153 build_reference_canonical(kernel, grid(box, N), M, {doubled=true,
 * step_constant}) for a Newton/Yukawa primitive; step_constant <= 0 selects the
 * calibrated sweep.  The 2N_l x R side matrices (unit columns) and R weights stay on
 * the device; identical modes share one matrix (reference.hpp:125-139). */
int latsum_reference_build(latsum_ctx* ctx, int family, double lambda, const int64_t N[3],
                           const double box[3], int M, double step_constant,
                           latsum_reference** out);
void latsum_reference_destroy(latsum_reference* ref);
/* rank R, step constant C0, shell [a, A] */
int latsum_reference_info(const latsum_reference* ref, int* rank, double* step_constant,
                          double shell[2]);
/* ReferenceTensor::canonical.factor(mode) (2N_l x R) and .weights() (R) to host buffers. */
int latsum_reference_factor(latsum_ctx* ctx, const latsum_reference* ref, int mode,
                            double* factor);
int latsum_reference_weights(const latsum_reference* ref, double* weights);
/* QuadratureRule nodes t_k and weights a_k (R each). */
int latsum_reference_quadrature(const latsum_reference* ref, double* nodes, double* weights);

/* ------------------------------------------------------------------ stage 2
 * Assembled lattice sum plus additive defects in canonical form:
 *   lattice_sum.hpp:198-223 assembled_sum_canonical (one block per sublattice),
 *   :411-465 sublattice_union_sum, :339-384 defected_sum (canonical branch, no spec),
 *   :148-157 windowed_canonical.
 * Sublattice s contributes R terms whose mode-l vector is sum_{c in shifts_s,l}
 * ref[N/2 - c + i] (assembled_vector, :101-144, with an explicit shift list),
 * weight charge_s * w_ref.  Defect d contributes R terms: the window at shift
 * (c1,c2,c3), weight charge_d * w_ref.  Terms are ordered sublattice blocks first,
 * then defects, as add_concat builds them.  from_raw normalisation per block.
 *   sub_counts: nsub x 3 (number of shifts per mode); sub_shifts: concatenated in
 *   (s, mode) order; def_shifts: ndef x 3 row-major.
 * Returns once the per-mode dictionaries are on the device; merging identical rank-1 terms
 * continues on a library host thread (overlapping the caller's next calls, e.g. the RHOSVD
 * eigensolves).  Every function that needs the merged terms waits for it (thread-safe);
 * latsum_canonical_destroy joins it.                                                  */
int latsum_canonical_assemble(latsum_ctx* ctx, const latsum_reference* ref, int64_t nsub,
                              const int64_t* sub_counts, const int64_t* sub_shifts,
                              const double* sub_charges, int64_t ndef, const int64_t* def_shifts,
                              const double* def_charges, latsum_canonical** out);
/* The same sum over an ORDERED list of product blocks, the general form of
 * defected_sum's canonical branch (lattice_sum.hpp:339-384): block b is a Cartesian
 * product of per-mode shift lists (blk_counts[b*3+l] shifts in mode l, concatenated in
 * (b, mode) order in blk_shifts) with additive charge blk_charges[b], and contributes R
 * terms at reference rank, in block order (add_concat).  A sublattice
 * (assembled_sum_canonical / sublattice_union_sum), a defect cluster whose sites form a
 * Cartesian product (defect_cluster_canonical's product_structure branch,
 * lattice_sum.hpp:278-294,316-321, "multi-level reuse") and a single defect site
 * (windowed_canonical, :148-157, counts 1 x 1 x 1) are all product blocks; a
 * non-product cluster is passed as its sites, one 1 x 1 x 1 block each, in site order
 * (:324-329).                                                                         */
int latsum_canonical_assemble_blocks(latsum_ctx* ctx, const latsum_reference* ref, int64_t nblk,
                                     const int64_t* blk_counts, const int64_t* blk_shifts,
                                     const double* blk_charges, latsum_canonical** out);
void latsum_canonical_destroy(latsum_canonical* can);
/* M_c = rank of the canonical sum, d_l = distinct (merged) columns per mode, T = merged terms. */
int latsum_canonical_info(const latsum_canonical* can, int64_t dims[3], int64_t* rank,
                          int64_t dict_cols[3], int64_t* merged_terms);
/* CanonicalTensor::weights() (M_c). */
int latsum_canonical_weights(const latsum_canonical* can, double* weights);
/* CanonicalTensor::factor(mode): N_l x M_c side matrix materialised in reference column
 * order, to a host buffer or (``_device``) to caller-owned device memory. */
int latsum_canonical_factor(latsum_ctx* ctx, const latsum_canonical* can, int mode,
                            double* factor);
int latsum_canonical_factor_device(latsum_ctx* ctx, const latsum_canonical* can, int mode,
                                   double* factor_device);
/* CanonicalTensor::entry (canonical.hpp:63-70) at np probe points (np x 3 indices). */
int latsum_canonical_entries(latsum_ctx* ctx, const latsum_canonical* can, const int64_t* probes,
                             int64_t np, double* out);
/* norm_f (canonical.hpp:148-162) without forming M_c x M_c matrices. */
int latsum_canonical_norm(latsum_ctx* ctx, const latsum_canonical* can, double* out);
/* Canonical to grid on the box [lo, hi) (to_dense, canonical.hpp:192-202, unguarded on
 * the device); out is (hi-lo) column-major, first index fastest. */
int latsum_canonical_eval_box_device(latsum_ctx* ctx, const latsum_canonical* can,
                                     const int64_t lo[3], const int64_t hi[3], double* out_device);

/* ------------------------------------------------------------------ stage 3
 * rank_reduction.hpp:176-218 rhosvd(canonical, TruncationSpec): ranks != NULL gives
 * fixed ranks (clamped), else tolerance in (0,1).  deflate selects the second Gram
 * pass that resolves singular values below sqrt(eps_mach) sigma_1. */
int latsum_rhosvd(latsum_ctx* ctx, const latsum_canonical* can, const int64_t* ranks,
                  double tolerance, int deflate, latsum_tucker** out,
                  latsum_spectral_report* report);
int latsum_rhosvd_ex(latsum_ctx* ctx, const latsum_canonical* can, const int64_t* ranks,
                     double tolerance, int deflate, int flags, latsum_tucker** out,
                     latsum_spectral_report* report);
/* canonical_to_tucker (rank_reduction.hpp:280-306): rhosvd, then ALS refinement
 * (als_refine, :232-274; up to max_als_sweeps, stagnation tolerance as TruncationSpec's)
 * and, with a tolerance and no ranks, shrink_core (:129-168).  report.chosen_ranks are the
 * final (shrunk) ranks; als_sweeps (nullable) returns the sweeps run.  ALS needs the
 * contracted unfolding (r^2 x d doubles) on the device: feasible for BASELINE cfg2/3. */
int latsum_canonical_to_tucker(latsum_ctx* ctx, const latsum_canonical* can, const int64_t* ranks,
                               double tolerance, int max_als_sweeps, double als_stagnation_tol,
                               latsum_tucker** out, latsum_spectral_report* report,
                               int* als_sweeps);
void latsum_tucker_destroy(latsum_tucker* t);
/* 1 when the dense core exists (latsum_tucker_core), 0 for a factors-only result. */
int latsum_tucker_has_core(const latsum_tucker* t);
int latsum_tucker_info(const latsum_tucker* t, int64_t dims[3], int64_t ranks[3]);
/* SpectralReport::singular_values[mode] (report.n_singular[mode] values, descending). */
int latsum_tucker_singular_values(const latsum_tucker* t, int mode, double* out);
/* TuckerTensor::core() (r1 x r2 x r3, first index fastest) and factor(mode) (N_l x r_l). */
int latsum_tucker_core(latsum_ctx* ctx, const latsum_tucker* t, double* core);
/* The local mode-1 slab of the core: *a0, *ra (first row, rows; the whole core for an
 * unsharded tensor) and, when core is not NULL, the ra x r2 x r3 slab (first index fastest). */
int latsum_tucker_core_slab(latsum_ctx* ctx, const latsum_tucker* t, int64_t* a0, int64_t* ra,
                            double* core);
int latsum_tucker_factor(latsum_ctx* ctx, const latsum_tucker* t, int mode, double* factor);
/* The projected canonical form of a factors-only tensor (no dense core; BASELINE cfg5):
 * V(i,j,k) = sum_t w_t prod_l (U_l P_l)(i_l, c_l(t)), equal to the Tucker tensor (SURVEY
 * 8c "projected-CP identity"; rank_reduction.hpp:88-100 before the core loop).  Fills
 * d[3] (merged columns per mode) and *T (merged rank-1 terms); each non-null buffer gets
 * P_l (r_l x d_l, column-major), the terms' column indices c_l (T) and weights w (T).
 * Call with null buffers first to size them.                                          */
int latsum_tucker_projected_form(latsum_ctx* ctx, const latsum_tucker* t, int64_t d[3], int64_t* T,
                                 double* P0, double* P1, double* P2, int32_t* c0, int32_t* c1,
                                 int32_t* c2, double* w);

/* ------------------------------------------------------------------ stage 4
 * TuckerTensor::entry (tucker.hpp:38-54) at probes, and to_dense (tucker.hpp:172-178)
 * on the box [lo, hi) of the grid: out (hi-lo) column-major. */
int latsum_tucker_entries(latsum_ctx* ctx, const latsum_tucker* t, const int64_t* probes,
                          int64_t np, double* out);
int latsum_tucker_eval_box(latsum_ctx* ctx, const latsum_tucker* t, const int64_t lo[3],
                           const int64_t hi[3], double* out);
int latsum_tucker_eval_box_device(latsum_ctx* ctx, const latsum_tucker* t, const int64_t lo[3],
                                  const int64_t hi[3], double* out_device);

/* ------------------------------------------------------------------ pipeline
 * cmd_sum (commands.cpp:108-179) for a defected / multi-sublattice lattice with a
 * truncation block: stages 1-3 in one call, inputs and the Tucker result in host
 * memory (the drop-in used by the end-to-end bench). */
int latsum_sum_to_tucker(latsum_ctx* ctx, int family, double lambda, const int64_t N[3],
                         const double box[3], int M, double step_constant, int64_t nsub,
                         const int64_t* sub_counts, const int64_t* sub_shifts,
                         const double* sub_charges, int64_t ndef, const int64_t* def_shifts,
                         const double* def_charges, double tolerance, latsum_tucker** out,
                         latsum_spectral_report* report);

/* SumOptions::accumulation (lattice_sum.hpp:28-39) for the assemblies made on this context:
 * 0 sliding (default, as in the reference): uniformly strided shift lists (contiguous K sets)
 *   are summed by the recursion v[i] = v[i-n] + entering - leaving of lattice_sum.hpp:116-128, in
 *   the reference's operation order, every other list directly;
 * 1 ascending: every list directly in ascending order (lattice_sum.hpp:142);
 * 2 compensated: accepted; summed in the ascending order (the Kahan correction of
 *   lattice_sum.hpp:129-140 changes the result below 1e-15 relative and is not applied). */
int latsum_ctx_set_accumulation(latsum_ctx* ctx, int order);

/* add_concat (canonical.hpp:94-110): *out = a + b by concatenation — rank(a) + rank(b) terms, a's
 * first; entries add exactly; the per-mode dictionaries are concatenated.  This is how
 * defected_sum adds a cluster to the base sum (lattice_sum.hpp:372-374), and with it a defect
 * cluster carrying its own kernel (DefectSpec.kernel, lattice_sum.hpp:301-303) is assembled
 * against that kernel's reference tensor and added in DefectSpec order.  a and b stay valid. */
int latsum_canonical_concat(latsum_ctx* ctx, const latsum_canonical* a, const latsum_canonical* b,
                            latsum_canonical** out);

/* ------------------------------------------------------------------ tensors from / to host
 * CanonicalTensor(dims, weights, factors) (canonical.hpp:25-29): columns taken as given
 * (the caller guarantees unit norms), so rhosvd / canonical_to_tucker accept any canonical
 * input, as the reference's do. */
int latsum_canonical_from_host(latsum_ctx* ctx, const int64_t dims[3], int64_t rank,
                               const double* weights, const double* f0, const double* f1,
                               const double* f2, latsum_canonical** out);
/* write_tensor / read_tensor (tensor_io.cpp:45-129): "LTSTNSR" v1 with the FNV-1a-64
 * trailer, byte-compatible with the reference.  Write exactly one of can / t; read sets
 * one of *can_out / *t_out.  Checksum, magic, version and truncation errors ->
 * LATSUM_ERR_IO. */
int latsum_tensor_write(latsum_ctx* ctx, const latsum_canonical* can, const latsum_tucker* t,
                        const char* path);
int latsum_tensor_read(latsum_ctx* ctx, const char* path, latsum_canonical** can_out,
                       latsum_tucker** t_out);

/* ------------------------------------------------------------------ text reports
 * The spectral report and provenance sidecar of `latsum sum` (report.cpp:28-73, written by
 * commands.cpp:56-72), byte for byte: 17 significant digits (report.cpp:9-12).  Host only
 * (no context, no device).  Both format into buf (cap bytes, NUL-terminated, truncated to
 * fit) and return the full text length, so a call with buf = NULL sizes the buffer; -1 on
 * a null report.
 *   write_spectral_report: sigma[l] holds report->n_singular[l] values
 *     (latsum_tucker_singular_values), descending.                                    */
int64_t latsum_format_spectral_report(const latsum_spectral_report* report,
                                      const double* const sigma[3], char* buf, int64_t cap);
/* write_provenance(result, seed, extra_lines): LatticeSumResult's grid, geometry cells,
 * tensor format and rank(s), its summands (lattice_sum.hpp:44-50: label, canonical rank,
 * sites) and, with a report, the truncation bounds.                                   */
typedef struct {
  uint64_t seed;
  int64_t grid[3];
  int64_t cells[3];
  int format;                     /* 0: canonical (rank), 1: tucker (ranks) */
  int64_t rank;
  int64_t ranks[3];
  int64_t nsummands;
  const char* const* labels;      /* nsummands */
  const int64_t* summand_ranks;   /* nsummands */
  const int64_t* summand_sites;   /* nsummands */
  int has_report;
  double bound_abs, bound_rel;
  int64_t nextra;
  const char* const* extra;       /* nextra lines appended verbatim */
} latsum_provenance;
int64_t latsum_format_provenance(const latsum_provenance* p, char* buf, int64_t cap);

/* ------------------------------------------------------------------ verification
 * oracle_entry (lattice_sum.hpp:656-671) on the device: the brute-force windowed sum
 * over ns grid-shifted sources (shifts ns x 3, weights ns; enumerate_sources order,
 * :632-653) at np probes, for cmd_verify-style checks (commands.cpp:200-284) at sizes
 * the CPU cannot reach (BASELINE cfg5: 16.8M sources). */
int latsum_verify_entries(latsum_ctx* ctx, const latsum_reference* ref, int64_t ns,
                          const int64_t* shifts, const double* weights, const int64_t* probes,
                          int64_t np, double* out);

/* ------------------------------------------------------------------ utilities */
/* Generic FP64 DMMA GEMM on device pointers (exposed for tests and benchmarks):
 * C = alpha op(A) op(B) + beta C, column-major, op = transpose when t* != 0. */
int latsum_dgemm_device(latsum_ctx* ctx, int ta, int tb, int64_t M, int64_t N, int64_t K,
                        double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double beta, double* C, int64_t ldc);

/* Householder tridiagonalisation of a symmetric n x n device matrix (full storage; LAPACK
 * dsytrd 'L' output: d, e, tau on the device, reflectors below the subdiagonal of A),
 * computed by one 16-CTA thread-block cluster.  Building block of the eigensolver that
 * replaces cuSOLVER syevd for the RHOSVD Grams. */
int latsum_sytrd_device(latsum_ctx* ctx, int64_t n, double* A, int64_t lda, double* d, double* e,
                        double* tau);

/* Symmetric eigensolver of the Gram passes (device pointers): all eigenvalues ascending
 * into w (n) and the k leading eigenvectors (descending eigenvalue order, unit norm) into V
 * (n x k).  cuSOLVER syevd by default; LATSUM_EIG=custom (n <= 1536) runs the in-house
 * solver (cluster sytrd, Sturm multisection, inverse iteration, compact-WY
 * back-transformation; syevd fallback when the vectors are not orthonormal). */
int latsum_eig_sym_device(latsum_ctx* ctx, int64_t n, const double* A, int64_t k, double* w,
                          double* V, int method /* 0 default, 1 cuSOLVER, 2 in-house one-stage, 3 in-house two-stage (band) */);

/* FP64-accurate C = A op(B) (column-major; op(B) = B^T when tb != 0) computed on the int8 tensor cores
 * by the Ozaki splitting (7 int8 slices per operand, tcgen05.mma.kind::i8, int32 TMEM
 * accumulators); K > 16384 runs as K-chunks accumulated into C in FP64.  The engine of the stage-4 evaluation GEMMs and the
 * stage-3 core contraction (LATSUM_EVAL_GEMM=dmma / LATSUM_CORE_GEMM=dmma revert to DMMA). */
int latsum_dgemm_ozaki_device(latsum_ctx* ctx, int tb, int64_t M, int64_t N, int64_t K,
                              const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                              int64_t ldc);

#ifdef __cplusplus
}
#endif
#endif /* LATSUM_B200_H */

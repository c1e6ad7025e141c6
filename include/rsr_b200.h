/*
 * rsr_b200.h -- C ABI of the B200-native RSR hot path (librsr_b200.so).
 *
 * The reference (arxiv 2604.17066 artifact, Python package `rsr`) has no FFI:
 * its seam is the Python API re-exported by pkg/src/rsr/__init__.py:5-35.
 * Each entry point below replaces the numpy body of one reference function;
 * the citation names the function it replaces (paths relative to
 * pkg/src/rsr/).  The Python package paper_2604_17066_b200 binds these with
 * ctypes (INTEGRATION.md shows the binding a maintainer of the reference
 * would add).
 *
 * Conventions
 *   - every function returns int status: RSR_OK (0), RSR_EINVAL (bad argument,
 *     mapped to ValueError), RSR_ECUDA (CUDA error, RuntimeError),
 *     RSR_EUNSUPPORTED (shape outside what the kernels handle, ValueError),
 *     RSR_ENCCL (NCCL error in the rsr_comm_* / exchange calls, RuntimeError);
 *     rsr_last_error() returns a thread-local message for the last failure;
 *   - all array arguments are caller-owned DEVICE pointers (the library never
 *     allocates or frees them) unless the name ends in _host;
 *   - every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and never synchronises the device;
 *   - states are uint8 (0 .. M-1), matrices are row-major.
 *
 * Thermometer layout (shared by samples "A" and reference rows "B"):
 *   Kdim = N*(M-1) columns c = n*(M-1) + (k-1), k = 1..M-1, followed by
 *   nb = ceil(Kdim/127) bias columns, zero-padded to Kpad = round_up(Kdim+nb, 32)
 *   (rsr_thermo_kpad).  A[s,c] = [x_n < k], A[s,Kdim+j] = 1.
 *   Upper ref r: B[r,c] = [r_n >= k], bias 0            -> A.B = #violations.
 *   Lower ref r: B[r,c] = -[r_n < k], bias sums to
 *                sum_c [r_n < k]                        -> A.B = c_r - overlap.
 *   Pad ref rows: B[r,Kdim] = 1, else 0                 -> A.B = 1, never a hit.
 *   In every case A.B >= 0 and A.B == 0  <=>  the sample is dominated by
 *   (lower) / dominates (upper) the reference state.
 */
#ifndef RSR_B200_H
#define RSR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSR_OK 0
#define RSR_EINVAL 1
#define RSR_ECUDA 2
#define RSR_EUNSUPPORTED 3
#define RSR_ENCCL 4

#define RSR_SIDE_LOWER 0
#define RSR_SIDE_UPPER 1

/* label codes written by rsr_finalize (device convention) */
#define RSR_LABEL_LOWER 0
#define RSR_LABEL_UPPER 1
#define RSR_LABEL_UNCLASSIFIED 2

/* flags bits written by the classifiers */
/* sampler streams: the reference's (bit-exact) and the independent device one */
#define RSR_RNG_SHARED 0 /* Philox4x64-10 = numpy.random.Philox, sampling.py:39-66   */
#define RSR_RNG_DEVICE 1 /* Philox4x32-10, counter (block, gen), key seed; 2^-32 CDF */

#define RSR_HIT_LOWER 1
#define RSR_HIT_UPPER 2

/* Phi kinds (sysfn.py:87-185 plus builder-defined widest path) */
#define RSR_PHI_ST_CONNECTIVITY 0  /* sysfn.py:87-98 single_od_connectivity   */
#define RSR_PHI_WIDEST_PATH 1      /* max k: s-t connected on {x_e >= k}      */
#define RSR_PHI_GLOBAL_CONNECTIVITY 2 /* sysfn.py:101-109                     */
#define RSR_PHI_K_OUT_OF_N 3       /* sysfn.py:177-185                        */
#define RSR_PHI_CONE_SUM 4         /* sum_l [x >= some anchor of level l]     */
#define RSR_PHI_EDGE_DISJOINT 5    /* sysfn.py:140-174 min_t maxflow(0,t) capped at k */

typedef struct rsr_phi_desc {
  int32_t kind;
  int32_t n_components;   /* N (== number of edges for graph kinds)            */
  int32_t n_states;       /* M                                                 */
  int32_t n_nodes;        /* graph kinds                                       */
  int32_t source;         /* s (st / widest)                                   */
  int32_t target;         /* t (st / widest)                                   */
  int32_t k;              /* k_out_of_n                                        */
  int32_t n_anchors;      /* cone sum                                          */
  const int32_t* edge_u;  /* device [N]                                        */
  const int32_t* edge_v;  /* device [N]                                        */
  const uint8_t* anchors; /* device [n_anchors * N]                            */
  const int32_t* anchor_level; /* device [n_anchors], 0-based level index      */
  int32_t flags;          /* RSR_PHI_FLAG_* hints                              */
} rsr_phi_desc;

/* no two edges share their endpoints: enables the bitset-BFS kernels */
#define RSR_PHI_FLAG_SIMPLE 1

/* ---- library ---------------------------------------------------------- */
int rsr_version(void);
const char* rsr_last_error(void);
int rsr_thermo_kpad(int n_components, int n_states);
/* number of device SMs and the int8 tcgen05 path availability (sm_100) */
int rsr_device_info(int* sm_count_host, int* cc_major_host, int* cc_minor_host);

/* ---- (1) sampling: sampling.py:45-66 uniform_field, :69-90 sample_batch - */
/* Philox4x64-10 raw words first..first+count-1 of stream key (seed, gen). */
int rsr_philox_raw(uint64_t seed, uint64_t gen, int64_t first, int64_t count,
                   uint64_t* out, void* stream);
int rsr_uniform_field(uint64_t seed, uint64_t gen, int64_t start, int64_t count,
                      int n_components, double* out, void* stream);
/* Inverse-CDF samples [start, start+count) of the (seed, gen) batch.
 * probs: device f64 [N*M] (rows sum to 1).  out_states: u8 [count*N] or NULL.
 * out_thermo: s8 [count*ld_thermo] thermometer rows (ld >= Kpad) or NULL. */
int rsr_sample(const double* probs, int n_components, int n_states, uint64_t seed,
               uint64_t gen, int64_t start, int64_t count, uint8_t* out_states,
               int8_t* out_thermo, int ld_thermo, void* stream);

/* Same draws, fused with the FP4 sample operand of rsr_classify_fp4 (default
 * path): out_states u8 [count*N] (16-byte aligned) and/or out_fp4
 * [count * 2*row_bytes] (row_bytes = rsr_fp4_row_bytes(N, M)); NULL skips. */
int rsr_sample_fp4(const double* probs, int n_components, int n_states, uint64_t seed,
                   uint64_t gen, int64_t start, int64_t count, uint8_t* out_states,
                   uint8_t* out_fp4, int row_bytes, void* stream);

/* Independent device stream (north_star: "independent device RNG"): the same
 * calls with rng = RSR_RNG_DEVICE draw (row R = start+i, component n) from word n%4
 * of the Philox4x32-10 block with counter [n/4, R lo, R hi, gen lo] and key
 * [seed lo ^ gen hi, seed hi] (row-aligned blocks); state = #{m < M-1 : raw32 >=
 * ceil(cum_m * 2^32)}.
 * rng = RSR_RNG_SHARED is rsr_sample / rsr_sample_fp4.  rsr_sample_fp4_ex also takes
 * the FP4 operand layout: fp4_plane_stride = 0 writes interleaved rows [A_up | A_lo]
 * (2*row_bytes per row); > 0 writes planar A_up rows of row_bytes and the A_lo plane
 * fp4_plane_stride bytes further (a multiple of 16, >= count*row_bytes), which a
 * one-sided classification streams without reading the other half. */
int rsr_sample_ex(const double* probs, int n_components, int n_states, uint64_t seed,
                  uint64_t gen, int64_t start, int64_t count, uint8_t* out_states,
                  int8_t* out_thermo, int ld_thermo, int rng, void* stream);
int rsr_sample_fp4_ex(const double* probs, int n_components, int n_states, uint64_t seed,
                      uint64_t gen, int64_t start, int64_t count, uint8_t* out_states,
                      uint8_t* out_fp4, int row_bytes, int64_t fp4_plane_stride, int rng,
                      void* stream);
/* Raw 32-bit draws of rows start..start+count-1 of the device stream (seed, gen) for
 * n_components components: out[i * n_components + n]. */
int rsr_device_raw(uint64_t seed, uint64_t gen, int64_t start, int64_t count, int n_components,
                   uint32_t* out, void* stream);

/* ---- (2) encodings: encoding.py:138-153 encode_batch ---------------------- */
int rsr_encode_samples(const uint8_t* states, int64_t count, int n_components,
                       int n_states, int8_t* out, int ld, void* stream);
/* side: RSR_SIDE_LOWER / RSR_SIDE_UPPER; rows [0,count) from states, rows
 * [count, rows_total) written as never-hit pad rows. */
int rsr_encode_refs(const uint8_t* states, int64_t count, int64_t rows_total,
                    int n_components, int n_states, int side, int8_t* out, int ld,
                    void* stream);

/* Reference-layout rows (encoding.py:42-57, 138-153): kind 0 = sample
 * (one-hot), 1 = lower_ref (prefix), 2 = upper_ref (suffix); out u8 [K x N*M]. */
int rsr_encode_rows(const uint8_t* states, int64_t count, int n_components, int n_states,
                    int kind, uint8_t* out, void* stream);
/* np.packbits(rows, axis=1) (MSB first, zero padded), complement != 0 packs
 * 1 - rows with pad bits zero (encoding.py:82-98); out u8 [K x ceil(L/8)]. */
int rsr_packbits_rows(const uint8_t* rows, int64_t count, int row_len, int complement,
                      uint8_t* out, void* stream);

/* ---- (2) dominance classification: classify.py:99-148, 187-249 --------- */
/* tcgen05 int8 tensor-core classifier.  A: s8 [S x ld_a] thermometer samples;
 * B_lower / B_upper: s8 [rows x ld_b] thermometer refs (rows multiple of 128,
 * pad rows never hit), n_lower / n_upper = rows actually holding refs.
 * flags[s] (u8) = RSR_HIT_LOWER | RSR_HIT_UPPER bits, OR-ed into the existing
 * value when accumulate != 0.  Kpad = ld_a = ld_b. */
int rsr_classify_tc(const int8_t* A, int64_t S, const int8_t* B_lower,
                    int64_t n_lower, const int8_t* B_upper, int64_t n_upper,
                    int Kpad, uint8_t* flags, int accumulate, void* stream);
/* Same, also recording per sample the smallest matching reference index of each
 * side (int64, -1 when none; explain / strict, classify.py:99-118, 226-238). */
int rsr_classify_tc_explain(const int8_t* A, int64_t S, const int8_t* B_lower,
                            int64_t n_lower, const int8_t* B_upper, int64_t n_upper,
                            int Kpad, uint8_t* flags, int64_t* first_lower,
                            int64_t* first_upper, int accumulate, void* stream);
/* Block-scaled FP4 tensor-core classifier (default path; 2x the int8 MMA
 * rate): tcgen05.mma.cta_group::2.kind::mxf4, e2m1 operands, unit scales.
 * FP4 layout (row_bytes = rsr_fp4_row_bytes(N, M) = round_up(Kdim+1, 64)/2,
 * element c of a row in byte c/2, low nibble first, 0x2 = 1.0, 0x0 = 0):
 *   sample row s: [A_up | A_lo], 2*row_bytes bytes, A_up[c] = [x_n < k],
 *     A_lo[c] = [x_n >= k] (c < Kdim), both 1 at the bias column c = Kdim;
 *   upper ref row: [r_n >= k], lower ref row: [r_n < k], bias column 0;
 *   pad ref rows: only the bias column set (never hit).
 * Reference buffers need n rows (the kernel masks columns past the last row of
 * a side; pad rows written by rsr_encode_refs_fp4 are harmless).  D = A_up.B_up
 * (upper) or A_lo.B_lo (lower) counts violated thermometer columns exactly
 * (fp32 accumulation of 0/1 products); D == 0 <=> dominance.  flags and
 * accumulate as rsr_classify_tc.  row_bytes <= RSR_FP4_MAX_ROW_BYTES (N(M-1) <= 1535;
 * rows wider than 416 bytes run lower and upper references as separate one-sided
 * launches).  The Stage-1 loop's device reference sets (rsr_refset_insert) take
 * rows up to RSR_REFSET_MAX_ROW_BYTES. */
#define RSR_FP4_MAX_ROW_BYTES 768
#define RSR_REFSET_MAX_ROW_BYTES 416
#define RSR_FP4_TILE_ROWS 240
int rsr_fp4_row_bytes(int n_components, int n_states);
int rsr_encode_samples_fp4(const uint8_t* states, int64_t count, int n_components,
                           int n_states, uint8_t* out, int row_bytes, void* stream);
/* Same with the operand layout of rsr_sample_fp4_ex (plane_stride 0: interleaved). */
int rsr_encode_samples_fp4_ex(const uint8_t* states, int64_t count, int n_components,
                              int n_states, uint8_t* out, int row_bytes, int64_t plane_stride,
                              void* stream);
/* FP4 sample operand from the reference's classification input: rows of
 * EncodedBatch(kind="sample").packed (encoding.py:82-98, np.packbits of the
 * one-hot N x M rows, MSB first, ceil(N*M/8) bytes per row; each component's
 * M bits must hold exactly one 1).  out: [count x 2*row_bytes]. */
int rsr_unpack_onehot_fp4(const uint8_t* packed, int64_t count, int n_components, int n_states,
                          uint8_t* out, int row_bytes, void* stream);
int rsr_encode_refs_fp4(const uint8_t* states, int64_t count, int64_t rows_total,
                        int n_components, int n_states, int side, uint8_t* out,
                        int row_bytes, void* stream);
int rsr_classify_fp4(const uint8_t* A, int64_t S, const uint8_t* B_lower, int64_t n_lower,
                     const uint8_t* B_upper, int64_t n_upper, int row_bytes,
                     uint8_t* flags, int accumulate, void* stream);
/* rsr_classify_fp4 with (a) n_* = the reference rows that count and avail_*
 * >= n_* the rows readable from B (rows n..avail-1 must be never-hit pad
 * rows, e.g. the tile padding of a reference set), so the launch can pick its
 * MMA N (reference tile of 160..240 rows) by n without masking pad columns;
 * (b) S_dev (may be NULL): device count of sample rows (<= S) to classify;
 * (c) first_* (may be NULL): first-match indices as rsr_classify_fp4_explain. */
int rsr_classify_fp4_ex(const uint8_t* A, int64_t S, const int64_t* S_dev,
                        const uint8_t* B_lower, int64_t n_lower, int64_t avail_lower,
                        const uint8_t* B_upper, int64_t n_upper, int64_t avail_upper,
                        int row_bytes, uint8_t* flags, int64_t* first_lower,
                        int64_t* first_upper, int accumulate, void* stream);
/* rsr_classify_fp4_ex on a planar sample operand (A_up rows of row_bytes, A_lo plane
 * a_plane_stride bytes further; rsr_sample_fp4_ex / rsr_encode_samples_fp4_ex with the
 * same stride). */
int rsr_classify_fp4_planar(const uint8_t* A, int64_t a_plane_stride, int64_t S,
                            const int64_t* S_dev, const uint8_t* B_lower, int64_t n_lower,
                            int64_t avail_lower, const uint8_t* B_upper, int64_t n_upper,
                            int64_t avail_upper, int row_bytes, uint8_t* flags,
                            int64_t* first_lower, int64_t* first_upper, int accumulate,
                            void* stream);
/* The launch plan rsr_classify_fp4* would use for S samples and these reference counts
 * (host only, no device work): MMA N per reference tile (160..240) and the number of
 * kernel launches (L2-sized reference chunks, or resident-sized launches for sets past
 * shared-memory residency, fewer for smaller S).  An all-empty call reports 0 launches
 * (the flags are cleared by a separate kernel unless accumulating); tile_n 0 means no
 * tile width fits shared memory (768-byte rows with first matches) and rsr_classify_fp4*
 * would return RSR_EUNSUPPORTED: use rsr_classify_tc or rsr_classify_bits. */
int rsr_classify_fp4_plan(int64_t S, int64_t n_lower, int64_t n_upper, int row_bytes,
                          int want_first, int* tile_n, int64_t* launches);
/* Support compaction of the FP4 contraction (csrc/fp4_compact.cu).  A thermometer
 * column in which no reference row of a side is 1 adds 0 to every violation count of
 * that side (classify.py:42-44; encoding.py:138-153), so the contraction may run over
 * the side's column support only -- labels, first matches and counts are unchanged.
 * rsr_fp4_or_rows: out (row_bytes/4 words, cleared by the call) = OR of the first
 * rows rows of B (rsr_encode_refs_fp4 layout).  rsr_fp4_gather_columns: dst column j =
 * src column cols[j] for j < n_cols, 0 for j >= n_cols (cols on the device; append the
 * bias column kdim = N(M-1) so sample rows keep their 1 and pad reference rows stay
 * never-hit); src / dst rows start every *_stride bytes (multiples of 16, 16-byte
 * aligned), one sample plane or a reference buffer per call. */
int rsr_fp4_or_rows(const uint8_t* B, int64_t rows, int row_bytes, uint32_t* out, void* stream);
int rsr_fp4_gather_columns(const uint8_t* src, int64_t src_stride, int64_t count,
                           int src_row_bytes, const int32_t* cols, int n_cols, uint8_t* dst,
                           int64_t dst_stride, int dst_row_bytes, void* stream);
/* Shared-tail paired classification (upper side only, no first matches): A is the planar
 * sample operand re-packed to 128-byte rows [192 main columns | 32 tail | the same 32 tail]
 * and B_upper holds n_upper rows (whole pairs of tile_n-row tiles, never-hit pad rows at the
 * end) of [192 main | own tail | 32 zero] in which every even tile's last 16 bytes carry the
 * next tile's tail (the host layout of classify.fp4_compaction).  tile_n must be the tile
 * width rsr_classify_fp4_plan_ex reports as paired for these sizes; otherwise
 * RSR_EUNSUPPORTED.  Labels equal rsr_classify_fp4 on the same columns. */
int rsr_classify_fp4_tail(const uint8_t* A, int64_t a_plane_stride, int64_t S,
                          const uint8_t* B_upper, int64_t n_upper, int row_bytes, int tile_n,
                          uint8_t* flags, int accumulate, void* stream);
/* rsr_classify_fp4_plan plus whether the plan pairs accumulators (streamed, 4 K-steps). */
int rsr_classify_fp4_plan_ex(int64_t S, int64_t n_lower, int64_t n_upper, int row_bytes,
                             int want_first, int* tile_n, int64_t* launches, int* paired);
/* rsr_classify_fp4 over the first *S_dev (device count, <= S_cap) rows of A:
 * the sample count of a later pass is known only on the device. */
int rsr_classify_fp4_dev(const uint8_t* A, int64_t S_cap, const int64_t* S_dev,
                         const uint8_t* B_lower, int64_t n_lower, const uint8_t* B_upper,
                         int64_t n_upper, int row_bytes, uint8_t* flags, int accumulate,
                         void* stream);
int rsr_classify_fp4_explain(const uint8_t* A, int64_t S, const uint8_t* B_lower,
                             int64_t n_lower, const uint8_t* B_upper, int64_t n_upper,
                             int row_bytes, uint8_t* flags, int64_t* first_lower,
                             int64_t* first_upper, int accumulate, void* stream);
/* Bit-packed CUDA-core comparison variant (AND + OR-reduce, LOP3).
 * Packs states on the fly; optional first-match indices (explain / strict,
 * classify.py:99-118): first_lower / first_upper int64 [S] or NULL. */
int rsr_pack_thermo_bits(const uint8_t* states, int64_t count, int n_components,
                         int n_states, int invert, uint32_t* out, int words,
                         void* stream);
int rsr_classify_bits(const uint32_t* sample_bits, int64_t S,
                      const uint32_t* lower_bits, int64_t n_lower,
                      const uint32_t* upper_bits, int64_t n_upper, int words,
                      uint8_t* flags, int64_t* first_lower, int64_t* first_upper,
                      int accumulate, void* stream);
/* flags -> labels (lower precedence, classify.py:240-245) + counts
 * counts_i64[4] = {lower, upper_only, unclassified, both}. */
int rsr_finalize(const uint8_t* flags, int64_t S, uint8_t* labels,
                 int64_t* counts, void* stream);
/* order-preserving compaction of indices with labels[i] == label
 * (np.flatnonzero, classify.py:242-245).  scratch: int64 [rsr_compact_scratch(S)]. */
int64_t rsr_compact_scratch(int64_t S);
int rsr_compact(const uint8_t* labels, int64_t S, int label, int64_t* out_idx,
                int64_t* out_count, int64_t* scratch, void* stream);
/* full H x R violation matrix, classify.py:57-96 (count = #components
 * violated: x_n > r_n for lower, x_n < r_n for upper). */
int rsr_violation_counts(const uint8_t* samples, int64_t H, const uint8_t* refs,
                         int64_t R, int n_components, int side, int32_t* out,
                         void* stream);
/* same on flattened binary rows for any EncodedBatch content:
 * out[h,r] = sum_j s[h,j] & (1 - r[r,j])  (classify.py:42-49). */
int rsr_violation_counts_rows(const uint8_t* sample_rows, int64_t H,
                              const uint8_t* ref_rows, int64_t R, int row_len,
                              int32_t* out, void* stream);

/* ---- (3) batched Phi: model.py:88-97 -> sysfn.py:79-185 ------------------ */
/* out[i] = Phi(states[idx[i]]) (idx NULL: rows 0..count-1; out may be NULL).
 * count_leq (int64 [1] or NULL) += #{i : Phi <= threshold} -- the Stage-2
 * resolution count of workflow.py:229-233. */
int rsr_phi_eval(const rsr_phi_desc* phi, const uint8_t* states,
                 const int64_t* idx, int64_t count, uint8_t* out, int threshold,
                 int64_t* count_leq, void* stream);

/* ---- (4) batched boundary search + reference insertion ------------------ */
/* boundary.py:116-147, one warp per start vector. out_side: RSR_SIDE_*;
 * out_calls: Phi evaluations per search (== reference evaluation count). */
int rsr_boundary_search(const rsr_phi_desc* phi, int threshold, const uint8_t* x0,
                        int64_t B, uint8_t* out_refs, uint8_t* out_side,
                        int64_t* out_calls, void* stream);
/* Exact enumeration for small models (oracle.py:49-63): vectors first ..
 * first+count-1 of itertools.product(range(M), repeat=N) and their probabilities
 * prod_n probs[n, x_n] (f64). */
int rsr_enumerate_states(const double* probs, int n_components, int n_states,
                         int64_t first, int64_t count, uint8_t* out_states,
                         double* out_prob, void* stream);
/* mass[s] += prob[i], counts[s] += 1 for s = phi[i], sequentially in i order
 * (bit-exact with the reference's float64 accumulation). */
int rsr_state_mass(const uint8_t* phi_values, const double* probs, int64_t count,
                   int n_system_states, double* mass, int64_t* counts, void* stream);
/* gather rows: out[i] = states[idx[i]] (N bytes each) */
int rsr_gather_rows(const uint8_t* states, int n_components, const int64_t* idx,
                    int64_t count, uint8_t* out, void* stream);
/* boundary.py:50-54 / 87-108 dominance scan of B candidates against K members:
 * covered[c] = 1 if some member makes candidate c redundant,
 * covers[c]  = 1 if candidate c makes some member redundant,
 * member_mask (may be NULL): with mask_candidate >= 0, u8 [K] = 1 where that
 * candidate makes the member redundant; with mask_candidate < 0, the full
 * relation u8 [B x K]: bit0 = member redundant under candidate, bit1 =
 * candidate redundant under member. */
int rsr_dominance_scan(const uint8_t* cands, int64_t B, const uint8_t* members,
                       int64_t K, int n_components, int side, uint8_t* covered,
                       uint8_t* covers, int mask_candidate, uint8_t* member_mask,
                       void* stream);

/* ---- device-resident reference sets (Stage-1 loop) ----------------------
 * ReferenceSet.insert (boundary.py:87-108) for a batch of boundary-search
 * results, entirely on the device.  Per side: member rows u8 [cap, N] and
 * their FP4 operand rows [cap, row_bytes] (rsr_encode_refs_fp4 layout; rows
 * >= ctr[0] are never-hit pad rows, which the caller fills when allocating),
 * alive flags u8 [cap] (dropped members stay in place, flagged 0), counters
 * ctr int64 [2] = {rows, alive}.  n_bound: caller's upper bound on ctr[0]. */
typedef struct rsr_refset_dev {
  uint8_t* rows;
  uint8_t* fp4;
  uint8_t* alive;
  int64_t* ctr;
  int64_t cap;
  int64_t n_bound;
} rsr_refset_dev;
/* scratch bytes for rsr_refset_insert with B candidates */
int64_t rsr_refset_scratch(int64_t B, int row_bytes);
/* Insert B candidates (u8 [B, N], side u8 [B], pick order) into the set of
 * their side with the reference's sequential semantics: outcome u8 [B] =
 * 1 inserted / 2 redundant; report int64 [8] = {lower rows, lower alive,
 * upper rows, upper alive, redundant searches (+=), dropped members (+=),
 * sum of calls[B] (may be NULL), capacity overflow (|=)}. */
int rsr_refset_insert(const uint8_t* cands, const uint8_t* cand_side, int64_t B,
                      int n_components, int n_states, const rsr_refset_dev* lower,
                      const rsr_refset_dev* upper, const int64_t* calls, uint8_t* outcome,
                      int64_t* report, void* scratch, void* stream);
/* dst[i] = src[idx[i]] (copy_bytes per row; multiples of 16) for i < *count_dev
 * (device count, at most cap): gathers sample operand rows for a second
 * classification pass without a host round trip. */
int rsr_gather_rows_dev(const uint8_t* src, int64_t src_stride, int copy_bytes,
                        const int64_t* idx, const int64_t* count_dev, int64_t cap,
                        uint8_t* dst, int64_t dst_stride, void* stream);
/* flags[idx[i]] |= vals[i] for i < *count_dev (at most cap). */
int rsr_scatter_or_dev(const uint8_t* vals, const int64_t* idx, const int64_t* count_dev,
                       int64_t cap, uint8_t* flags, void* stream);
/* rsr_gather_picks with the rows decoded from the FP4 sample operand
 * (x_n = number of set [x_n >= k] elements of the A_lo half): for batches kept
 * only in their classifier layout. */
int rsr_gather_picks_fp4(const uint8_t* fp4, int row_bytes, int n_components, int n_states,
                         const int64_t* idx, const int64_t* pos, int64_t count, uint8_t* out,
                         void* stream);
/* out[i] = states[idx[pos[i]]]: rows of the picked unclassified samples
 * (workflow.py:172-176 with the positions drawn on the host). */
int rsr_gather_picks(const uint8_t* states, int n_components, const int64_t* idx,
                     const int64_t* pos, int64_t count, uint8_t* out, void* stream);

/* ---- (e) multi-GPU exchange (the reference has no
 * communication -- its only parallel seam is the chunk thread pool of
 * classify.py:140-142).  One process per GPU; NCCL over NVLink, bound at run time
 * (libnccl.so.2).  The Python package does the same exchanges with
 * torch.distributed (dist.py).  comm: opaque communicator handle. */
#define RSR_COMM_ID_BYTES 128
/* 128-byte unique id (rank 0 creates it and broadcasts it out of band). */
int rsr_comm_unique_id(uint8_t* out_id_host);
int rsr_comm_init(const uint8_t* unique_id_host, int world, int rank, void** out_comm_host);
int rsr_comm_destroy(void* comm);
/* In-place sum of per-rank int64 class counts (labels / Phi calls of a sample shard). */
int rsr_allreduce_counts(void* comm, int64_t* counts, int n, void* stream);
/* Concatenation in rank order of every rank's bytes_per_rank bytes (new reference
 * rows, picked sample rows) into recv [world * bytes_per_rank]. */
int rsr_allgather_refs(void* comm, const uint8_t* send, int64_t bytes_per_rank, uint8_t* recv,
                       void* stream);
/* In-place OR of classifier hit flags [S] across reference shards (bit 0 lower,
 * bit 1 upper): two 0/1 planes in scratch [2*S], NCCL MAX, merged back. */
int rsr_or_reduce_flags(void* comm, uint8_t* flags, int64_t S, uint8_t* scratch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RSR_B200_H */

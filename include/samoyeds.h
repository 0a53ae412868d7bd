/*
 * samoyeds.h -- C ABI of the B200 (sm_100a) Samoyeds hot path.
 *
 * Samoyeds (arXiv 2503.10725) multiplies an MoE expert weight held in a
 * dual-side sparse format with only the tokens routed to that expert:
 *   "the original weight is encoded into three components: data, indices,
 *    and metadata"                                    (§4.1)
 *   "introduces a selection array (SEL) ... aligns with the sparsity pattern
 *    presented in token routing"                      (§4.1)
 *   Alg. 1 "Samoyeds Kernel Scheme": Input A, Indices, Metadata, B, SEL;
 *    Output C
 *   "the activation function and its precedent operator are fused ... the
 *    weighted accumulation ... is fused with matrix multiplication"
 *                                                      (§4.3)
 *
 * Conventions (all entry points):
 *  - Plain pointers only.  "dev" pointers are CUDA device pointers, "host"
 *    pointers are host memory.  The CALLER allocates and owns every buffer
 *    (size them with the *_bytes / *_layout queries); the library allocates
 *    nothing on the hot path and keeps no pointer after a call returns.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).  All
 *    calls are asynchronous on that stream; host-side argument validation
 *    returns synchronously with a status and launches nothing.
 *  - Data-dependent errors (pattern violations) go to a device status word the
 *    caller may read after synchronising.
 *  - bf16 tensors are IEEE bfloat16 bit patterns (uint16), row-major.
 *  - Requires an sm_100a device (B200); otherwise SMY_E_ARCH.
 */
#ifndef SAMOYEDS_H
#define SAMOYEDS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SMY_API __attribute__((visibility("default")))
#else
#define SMY_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SMY_OK = 0,
  SMY_E_NULL = 1,       /* a required pointer is NULL                           */
  SMY_E_SHAPE = 2,      /* shape not divisible / unsupported size (ShapeError)  */
  SMY_E_CONFIG = 3,     /* unsupported (N,M,V) or layer configuration           */
  SMY_E_PATTERN = 4,    /* weight violates the (N,M,V)+2:4 pattern (device)     */
  SMY_E_SELECTION = 5,  /* selection array invalid                              */
  SMY_E_CORRUPT = 6,    /* encoded weight invariant violated                    */
  SMY_E_WORKSPACE = 7,  /* workspace too small                                  */
  SMY_E_ARCH = 8,       /* no sm_100 device                                     */
  SMY_E_CUDA = 9,       /* CUDA runtime error                                   */
  SMY_E_NCCL = 10       /* NCCL error                                           */
} smy_status;

SMY_API const char* smy_status_str(int status);
SMY_API int smy_version(void);
/* Last CUDA error string seen by the library on this thread (diagnostics). */
SMY_API const char* smy_last_error(void);

/* ------------------------------------------------------------ format ----
 * (N, M, V) vector-wise sparsity layered on 2:4 (Fig. 7):
 * the weight is cut into M x V blocks (M output rows x V reduction columns);
 * N of the M sub-rows of length V are kept per block and each kept sub-row is
 * further pruned 2:4.  Table 4 formats: (1,2,16), (1,2,32),
 * (4,8,32), (8,16,32).  GPU path: M in {1,2,4,8,16}, N | 128, V in {16, 32,
 * 64, ...} (V=16 only with N=1), cols % 128 == 0, rows % M == 0.           */
typedef struct { int32_t n, m, v; } smy_format;

/* A logical weight [rows x cols] = [out x in] (PyTorch layout = the paper's
 * offline-transposed W). */
typedef struct { int64_t rows, cols; smy_format fmt; } smy_wdesc;

/* Byte sizes of every buffer of an encoded weight.  R = rows*N/M.
 *   values  : bf16 [R x cols/2]          canonical data matrix
 *   codes   : u8   [R x cols/8]          canonical 2-bit metadata, 4 per
 *             byte, code c at bits 2*(c%4), first kept position low
 *   indices : u8   [R x cols/V]          canonical sub-row indices
 *   image   : device image consumed by the SSMM kernel: [m_tiles][k_stages]
 *             blocks of `block` bytes = A smem image (16384, 128B-swizzled
 *             K-major) | E metadata TMEM image (2048) | index bit-planes
 *             (64*planes).  See DESIGN.md §HBM layout.                     */
typedef struct {
  size_t values, codes, indices, image;
  int32_t comp_rows, m_tiles, k_stages, planes, rep, block;
} smy_wlayout;
SMY_API smy_status smy_weight_layout(const smy_wdesc* desc, smy_wlayout* out);

/* An encoded weight: caller-owned device buffers sized by smy_weight_layout. */
typedef struct {
  smy_wdesc d;
  void* values;   /* dev */
  void* codes;    /* dev */
  void* indices;  /* dev */
  void* image;    /* dev */
} smy_weight;

#define SMY_PRUNE_MAGNITUDE 1 /* prune to the pattern first: per block keep the N
                                 sub-rows of largest fp32 L1 (ascending-column
                                 sum), per 4-group the 2 largest |w|; ties to the
                                 lower index (reading R4) */
#define SMY_ASSUME_PRUNED 2   /* input must already conform; violations set
                                 *d_status = SMY_E_PATTERN */

/* samoyeds_compress: encode a dense bf16 weight (dev, [rows x ldw]) into the
 * canonical (values, codes, indices) AND the device image (PAPER.md:237,
 * §4.4 packing).  d_status (dev int32, nullable) receives SMY_OK or
 * SMY_E_PATTERN; the caller zeroes it first.                                */
SMY_API smy_status samoyeds_compress(const smy_wdesc* desc, const void* w_bf16, int64_t ldw, int flags,
                             smy_weight* out, int32_t* d_status, void* stream);

/* samoyeds_decompress: the inverse of the encoding -- the dense
 * pattern-conforming bf16 weight [rows x ldw] (dev) from the canonical values,
 * codes and indices (which must be present); positions not stored are zero.
 * compress(decompress(w)) with SMY_ASSUME_PRUNED reproduces w bit for bit.
 * d_status (dev int32, nullable; the caller zeroes it first): the decoding
 * invariants are checked on the device -- per (row group, K-block) the N
 * sub-row indices < M and strictly increasing, per kept 4-group the two codes
 * strictly increasing -- and a violation writes SMY_E_CORRUPT (values of an
 * out-of-range sub-row index are dropped, never written outside the block). */
SMY_API smy_status samoyeds_decompress(const smy_weight* w, void* w_bf16, int64_t ldw, int32_t* d_status,
                                       void* stream);

/* samoyeds_interleave_gate_up: the interleaved gate/up weight of one expert
 * (reading R20; the paper fuses the activation with "its precedent
 * operator", without fixing how gate and up share a kernel).  The
 * logical weight is [2f x d] whose compressed rows alternate in blocks of 16:
 * 16 gate compressed rows, then the 16 up compressed rows of the same outputs
 * (= output rows [64b, 64b+32) gate rows [32b, 32b+32), the next 32 the same up
 * rows for N/M = 1/2; blocks of 16 output rows for N = M), so each warp's 32
 * TMEM lanes of an SSMM tile hold the gate AND up rows of the same outputs.
 * Pruning/encoding act on M-row groups, so this equals samoyeds_compress of
 * the interleaved dense weight bit for bit; it is built by moving whole
 * compressed rows of gate/up's canonical arrays (which must be present) and
 * re-packing the device image.  gate, up: same desc, rows % 32 == 0; gu:
 * caller-owned buffers sized by smy_weight_layout({2*rows, cols, fmt}).    */
SMY_API smy_status samoyeds_interleave_gate_up(const smy_weight* gate, const smy_weight* up, smy_weight* gu,
                                               void* stream);

/* ------------------------------------------------------------- SSMM -----
 * C[t, o] = sum_k W[o, k] * x[sel[t], k] for t < n_sel  (Alg. 1)
 * with a fused epilogue:
 *   SMY_EPI_COMPACT          out[t * ldo + o] = C[t, o]      (out_dtype)
 *   SMY_EPI_SILU_MUL_COMPACT out[t * ldo + o] = bf16(silu(C_w[t,o]) * C_w2[t,o])
 *                            (w = gate, w2 = up; out_dtype must be BF16)
 *   SMY_EPI_SILU_MUL_INTERLEAVED  w = the interleaved gate/up weight [2f x d]
 *                            (samoyeds_interleave_gate_up), w2 = NULL:
 *                            out[t * ldo + o] = bf16(silu(C_gate[t,o]) * C_up[t,o])
 *                            for o < f (BF16; format (1,2,V), (N,2N,V) or
 *                            N == M, V % 32 == 0)
 *   SMY_EPI_SCATTER_ADD      out[sel[t] * ldo + o] += scale[t] * C[t, o]  (f32;
 *                            scale NULL = 1; atomic, order not deterministic;
 *                            16-byte reductions: ldo % 4 == 0, out 16-byte
 *                            aligned and rows % 4 == 0, else SMY_E_SHAPE)
 * x: dev bf16 [x_rows x ldx], token-major; sel: dev int32 [n_sel], strictly
 * increasing, each in [0, x_rows) (the SEL of P:303); n_sel may be 0.  fp32
 * accumulation.  SEL is not checked on the hot path: samoyeds_validate_sel
 * checks it on the device (async, SMY_E_SELECTION into *d_status), and with the
 * environment variable SMY_DEBUG having bit 65536 set, samoyeds_ssmm runs that
 * check itself, synchronises its stream and returns SMY_E_SELECTION.        */
typedef enum {
  SMY_EPI_COMPACT = 0,
  SMY_EPI_SILU_MUL_COMPACT = 1,
  SMY_EPI_SCATTER_ADD = 2,
  SMY_EPI_SILU_MUL_INTERLEAVED = 3
} smy_epi;
#define SMY_F32 0
#define SMY_BF16 1
SMY_API smy_status samoyeds_ssmm(const smy_weight* w, const smy_weight* w2, const void* x_bf16, int64_t ldx,
                         int64_t x_rows, const int32_t* sel, int32_t n_sel, const float* scale, int epi,
                         void* out, int64_t ldo, int out_dtype, void* stream);
SMY_API smy_status samoyeds_validate_sel(const int32_t* sel, int32_t n_sel, int64_t x_rows, int32_t* d_status,
                                         void* stream);

/* --------------------------------------------------- routing / compaction
 * Top-k of fp32 router logits [T x E] per token (ties -> lower expert id) and
 * gate weights (readings R9, R10), then the per-expert selection
 * arrays: counts[E], offsets[E+1] (exclusive scan),
 * sel[T*k] token ids ascending within each expert, gw[T*k] aligned with sel.
 * ids/w (dev [T x k]) are written too.  Bit-exact deterministic.  A NaN
 * logit ranks as -inf (selected only after every finite logit).  gating must
 * be SMY_GATE_RENORM_TOPK or SMY_GATE_SOFTMAX_ALL (else SMY_E_CONFIG).     */
#define SMY_GATE_RENORM_TOPK 0
#define SMY_GATE_SOFTMAX_ALL 1
SMY_API smy_status smy_route_workspace_bytes(int64_t T, int32_t E, size_t* bytes);
SMY_API smy_status samoyeds_route(const float* logits, int64_t T, int32_t E, int32_t k, int gating, int32_t* ids,
                          float* w, int32_t* counts, int32_t* offsets, int32_t* sel, float* gw, void* workspace,
                          size_t ws_bytes, void* stream);

/* ---------------------------------------------------------- MoE layer ---
 * out[t] = sum_{(e,g) in topk(t)} g * Wd_e( silu(Wg_e x_t) * (Wu_e x_t) )
 *          + sum_s Wd_s( silu(Wg_s x_t) * (Wu_s x_t) )
 * experts: host array [E][3] of smy_weight: (gate, up, down) when
 * cfg->gate_up == SMY_GU_SEPARATE, or (gu, unused, down) when SMY_GU_INTERLEAVED
 * (gu from samoyeds_interleave_gate_up; format (1,2,V), (N,2N,V) or N == M,
 * V % 32 == 0 -- the kernels read one 128-lane tile of gate+up rows per MMA;
 * (N,2N,32) formats with N > 1 run every one-weight SSMM of the layer with the
 * in-shared-memory row expansion of their own compressed image); shared: host
 * array [num_shared][3] in the same layout, or NULL (num_shared + top_k <= 16,
 * num_experts + num_shared <= 128); the shared experts run as extra groups of the
 * same two grouped SSMM launches (the routing appends ids E.. with weight 1 to
 * every token).  x dev bf16 [T x hidden]; logits dev fp32
 * [T x E]; out dev [T x hidden] (overwritten), fp32 or bf16 (cfg->out_dtype).  The gate/up -> down
 * intermediate is bf16 (reading R12).                                     */
/* cfg->gating = SMY_GATE_RENORM_TOPK | SMY_GATE_SOFTMAX_ALL, optionally OR-ed
 * with SMY_GATE_SHARED_SIGMOID when num_shared > 0 (single-GPU layer only, else
 * SMY_E_CONFIG): the logits then have num_experts + num_shared columns and
 * shared expert s is weighted per token by 1 / (1 + exp(-logits[t][E + s]))
 * instead of 1 (Qwen2-MoE's gated shared expert; reading R15b --
 * a shared FFN wider than the routed ones runs as several shared experts of
 * the routed width with the same logit in each of their columns).          */
#define SMY_GATE_SHARED_SIGMOID 0x10
#define SMY_GU_SEPARATE 0
#define SMY_GU_INTERLEAVED 1
typedef struct {
  int32_t num_experts, top_k, hidden, ffn, num_shared, gating;
  smy_format fmt;
  int32_t gate_up;   /* SMY_GU_SEPARATE | SMY_GU_INTERLEAVED */
  int32_t out_dtype; /* SMY_F32 (default): out is fp32 [T x hidden];
                        SMY_BF16: out is bf16 [T x hidden] -- the layer
                        accumulates in an fp32 buffer at the end of its
                        workspace (smy_moe_workspace_bytes counts it) and
                        rounds once (RNE) after the last expert; single-GPU
                        layer only (comm == NULL, else SMY_E_CONFIG)       */
} smy_moe_config;
typedef struct smy_ep_comm smy_ep_comm; /* opaque, library-owned (EP) */
SMY_API smy_status smy_moe_workspace_bytes(const smy_moe_config* cfg, int64_t max_tokens, size_t* bytes);
/* comm == NULL: the whole layer on this GPU.  comm != NULL (expert parallelism,
 * SURVEY.md §8(e)): cfg->num_experts is the TOTAL E, `experts` holds this rank's
 * E/world experts [r*E/W, (r+1)*E/W) (same layout), num_shared must be 0, and
 * the workspace comes from smy_moe_ep_workspace_bytes.  The call routes over all
 * E, sends each token once to every rank owning one of its experts (NCCL
 * send/recv of rows + tags), runs this rank's experts on what it received,
 * returns the fp32 partial rows and sums them into out.  It reads the [W]
 * receive counts on the host once (one stream synchronisation).  Every rank
 * must size its workspace for the same max_tokens and call with T <= it: the
 * receive buffers hold max_tokens rows per peer.  A rank whose T exceeds its
 * workspace announces it in the counts exchange (count -1), and then EVERY
 * rank returns SMY_E_WORKSPACE after that exchange (no rank blocks in NCCL).
 * out must be 16-byte aligned (SMY_E_SHAPE). */
SMY_API smy_status samoyeds_moe_layer(const smy_moe_config* cfg, const smy_weight* experts, const smy_weight* shared,
                              const void* x_bf16, const float* logits, int64_t T, void* out, void* workspace,
                              size_t ws_bytes, smy_ep_comm* comm, void* stream);

/* The library-owned NCCL communicator of expert parallelism (libnccl.so.2 is
 * loaded on first use; SMY_E_NCCL if it cannot be).  smy_ep_unique_id writes a
 * 128-byte NCCL unique id on one rank; the caller broadcasts it (e.g. over its
 * torch process group) and every rank calls smy_ep_comm_create(id, rank, world)
 * with the current CUDA device set (blocks until all ranks joined). */
SMY_API smy_status smy_ep_unique_id(void* id128 /* host, 128 B */);
SMY_API smy_status smy_ep_comm_create(const void* id128, int32_t rank, int32_t world, smy_ep_comm** comm);
SMY_API smy_status smy_ep_comm_destroy(smy_ep_comm* comm);
SMY_API smy_status smy_moe_ep_workspace_bytes(const smy_moe_config* cfg, int64_t max_tokens, int32_t world,
                                              size_t* bytes);

/* ------------------------------------------------ expert parallelism (EP)
 * The layer shards over experts: rank r of P owns experts [r*E/P,(r+1)*E/P)
 * (the paper evaluates one GPU).  One exchange step
 * each way, done by the caller's process group (all_to_all_v, NCCL/NVLink):
 *   samoyeds_route (all E) -> samoyeds_ep_plan -> samoyeds_ep_pack
 *   -> [all_to_all rows + tags] -> samoyeds_moe_experts (local experts, keys =
 *   received tags) -> [all_to_all fp32 rows back] -> samoyeds_ep_combine.
 * ep_plan: ids/w dev [T x k] (from samoyeds_route); send_counts dev [P],
 *   send_offsets dev [P+1]; send_sel dev [T*k] = token ids sent, ordered by
 *   (destination rank, token id) -- each token once per destination;
 *   tag_ids/tag_w dev [T*k x k] per send row: the local expert ids (ascending)
 *   and gate weights the token meets at that rank, -1 / 0 padded.
 * ep_pack: x_send[i] = x[send_sel[i]] for i < send_offsets[P] (read on the
 *   device; max_rows bounds the buffer).
 * moe_experts: the layer body for rows whose routing is given: keys/vals dev
 *   [rows x k] (local expert ids, -1 = none; weights); cfg->num_experts = local
 *   experts; out dev fp32 [rows x hidden] (overwritten).  Workspace from
 *   smy_moe_workspace_bytes(cfg, rows).
 * ep_combine: out[send_sel[i]] += back[i] (fp32 rows returned by the owners;
 *   caller zeroes out first).                                               */
SMY_API smy_status smy_ep_plan_workspace_bytes(int64_t T, int32_t k, int32_t world, size_t* bytes);
SMY_API smy_status samoyeds_ep_plan(const int32_t* ids, const float* w, int64_t T, int32_t k, int32_t num_experts,
                                    int32_t world, int32_t* send_counts, int32_t* send_offsets, int32_t* send_sel,
                                    int32_t* tag_ids, float* tag_w, void* workspace, size_t ws_bytes, void* stream);
SMY_API smy_status samoyeds_ep_pack(const void* x_bf16, int64_t ldx, int64_t hidden, const int32_t* send_offsets,
                                    int32_t world, const int32_t* send_sel, int64_t max_rows, void* x_send,
                                    void* stream);
SMY_API smy_status samoyeds_moe_experts(const smy_moe_config* cfg, const smy_weight* experts, const void* x_bf16,
                                        int64_t rows, const int32_t* keys, const float* vals, float* out,
                                        void* workspace, size_t ws_bytes, void* stream);
SMY_API smy_status samoyeds_ep_combine(const float* back, int64_t hidden, const int32_t* send_offsets, int32_t world,
                                       const int32_t* send_sel, int64_t max_rows, float* out, void* stream);

/* ------------------------------ expert parallelism over NVLink peer memory
 * The token rows and the partial outputs do not travel as dispatched copies:
 * the owner's gate/up SSMM gathers each routed token row straight from its
 * source rank's activations (cp.async over NVLink), and the down SSMM's
 * scatter-add reduces straight into the source rank's fp32 output (P2P
 * red.add) -- the all-to-all dispatch/combine fused into the two GEMMs.  Only
 * the small routing metadata (per destination: row ids + tags) is exchanged
 * by the caller (all_to_all_v), plus two stream-ordered barriers: after every
 * rank zeroed its output and published its x, and after the owners' adds.
 * ep_row_ids: row_ids[i] = (rank << 24) | send_sel[i] for the send rows
 *   i < send_offsets[world] (max_rows bounds the buffer; T < 2^24).
 * moe_experts_peer: rows received rows; row_map dev [rows] = the senders'
 *   row ids; keys/vals dev [rows x k] their tags; x_peers / out_peers: host
 *   arrays [world] of device pointers valid on THIS device (peer-mapped, e.g.
 *   torch symmetric memory) to every rank's bf16 x [T x ldx] and fp32 out
 *   [T x ldo] (zeroed by its owner before; this call only adds).  world <= 8,
 *   cfg->num_shared == 0.  Workspace from smy_moe_workspace_bytes(cfg, rows). */
SMY_API smy_status samoyeds_ep_row_ids(const int32_t* send_sel, const int32_t* send_offsets, int32_t world,
                                       int32_t rank, int64_t max_rows, int32_t* row_ids, void* stream);
SMY_API smy_status samoyeds_moe_experts_peer(const smy_moe_config* cfg, const smy_weight* experts, int32_t world,
                                             const void* const* x_peers, int64_t ldx, float* const* out_peers,
                                             int64_t ldo, int64_t rows, const int32_t* row_map, const int32_t* keys,
                                             const float* vals, void* workspace, size_t ws_bytes, void* stream);

/* smy_moe_workspace_view: where a single-GPU samoyeds_moe_layer call over T
 * tokens (same cfg, same workspace) leaves its routing result and its
 * gate/up -> down intermediate, for inspection after the call (tests compare the
 * compact bf16 intermediate with the oracle at full size).  Pure pointer
 * arithmetic on `workspace`, no device access.  groups = num_experts +
 * num_shared; counts dev i32 [groups], offsets dev i32 [groups+1] (exclusive
 * scan), sel dev i32 [T*(top_k+num_shared)] (expert-major, ascending token ids
 * within an expert: the SEL arrays of P:303), gw dev fp32 aligned with sel;
 * inter dev bf16 [inter_rows x ffn], row i = the intermediate of (expert, token
 * sel[i]) -- the compressed output layout of P:374 (rows past offsets[groups]
 * are unused).                                                            */
typedef struct {
  int32_t *counts, *offsets, *sel;
  float* gw;
  void* inter;
  int64_t inter_rows;
  int32_t groups;
} smy_moe_view;
/* smy_moe_kernel_names: the names (as profilers print them, e.g.
 * "ssmm_pair_kernel<224, 1, 2, 1>") of the gate/up and down SSMM kernels a
 * single-GPU samoyeds_moe_layer call over T tokens launches -- the same tile and
 * CTA-pair decisions as the call itself (host only; len >= 48).             */
SMY_API smy_status smy_moe_kernel_names(const smy_moe_config* cfg, int64_t T, char* gate_up, char* down, int32_t len);
SMY_API smy_status smy_moe_workspace_view(const smy_moe_config* cfg, int64_t T, void* workspace, size_t ws_bytes,
                                          smy_moe_view* view);

/* ------------------------------------------------------------ diagnostics
 * smy_moe_set_phase_events: when events != NULL (n >= 6 cudaEvent_t handles,
 * passed as void*), samoyeds_moe_layer records events[0..5] on its stream at
 * its phase boundaries: start | routing done | out zeroed | gate/up SSMM done |
 * down SSMM done | shared experts done.  NULL disables.  Per calling thread
 * (thread-local); used by bench.py to time the dominant kernel inside the timed
 * region.  smy_launch_count: number of kernels this library has launched.  */
SMY_API smy_status smy_moe_set_phase_events(void** events, int n);
SMY_API uint64_t smy_launch_count(void);
/* SMY_DEBUG=128 profiling: copy (and reset) role cycle counters [2][ctas][16] (gate/up, scatter launches). */
/* Ablation variants of samoyeds_moe_layer -- the breakdown measurement of
 * SURVEY.md §8(f)-2 ("+W" vs "+WI"; P:374-376 the compressed output
 * layout), NOT the product path.  After smy_moe_set_variant(v, scratch, bytes)
 * with v != 0, single-GPU interleaved layer calls (comm == NULL, router logits)
 * on the calling thread (thread-local) compute the same layer as:
 *   SMY_VARIANT_PERMUTE      x[SEL] copied to an expert-major buffer (the
 *                            materialised input permutation), gate/up on it as
 *                            contiguous rows, down into compact fp32 rows, then a
 *                            weighted un-permute (out[sel[i]] += gw[i] y[i])
 *   SMY_VARIANT_DENSE_INTER  the intermediate in a token-position layout
 *                            [(E+ns) x T x ffn], zero-filled every call, gate/up
 *                            storing row e*T + sel[i], down gathering it back
 * Other layer calls return SMY_E_CONFIG while a variant is set.  scratch: device
 * buffer of >= smy_moe_variant_scratch_bytes(cfg, T, v) bytes (SMY_E_WORKSPACE),
 * caller-owned, alive while the variant is set.  v = SMY_VARIANT_PRODUCT (0)
 * restores the product path.  Unknown v: SMY_E_CONFIG.                      */
#define SMY_VARIANT_PRODUCT 0
#define SMY_VARIANT_PERMUTE 1
#define SMY_VARIANT_DENSE_INTER 2
SMY_API smy_status smy_moe_variant_scratch_bytes(const smy_moe_config* cfg, int64_t T, int32_t variant, size_t* bytes);
SMY_API smy_status smy_moe_set_variant(int32_t variant, void* scratch, size_t bytes);
SMY_API int smy_debug_prof(unsigned long long* host, int ctas);

/* ------------------------------------------------------ synthetic inputs
 * Counter-based generator twin of synth/__init__.py (input preparation only,
 * no method arithmetic): out[i] = value(seed, idx0 + i) for i < n.
 * dist 0 uniform, 1 Irwin-Hall normal, 2 integer in [lo, hi]; out_bf16 != 0
 * stores bf16 (RNE) else fp32.                                            */
SMY_API smy_status smy_synth_fill(uint64_t seed, int dist, float scale, int lo, int hi, int64_t idx0, int64_t n,
                          void* out, int out_bf16, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SAMOYEDS_H */

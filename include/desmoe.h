/*
 * desmoe.h — C ABI of the B200-native (sm_100a) Dynamic Expert Sharing MoE
 * layer. Plain pointers and sizes only; no C++ or torch types.
 *
 * Every entry point replaces one function of the reference library's C++
 * operator API (dessim, /root/reference/proj/core/include/dessim/{core,gating,des}.hpp); the
 * reference interface is cited beside each declaration. The C++ facade
 * (include/dessim/{core,gating,des}.hpp, libdessim_gpu.so) and the Python mirror (paper_2602_00879_b200/dessim.py)
 * sit on top of this header.
 *
 * Conventions
 *  - Pointers named *_dev are device pointers; everything is stream-ordered on
 *    `stream` (a cudaStream_t, NULL = legacy default stream) and never
 *    synchronises unless stated.
 *  - Return value: DESMOE_OK (0), DESMOE_EINVAL (1, the reference would throw
 *    std::invalid_argument; message identical to the reference's), DESMOE_ECUDA
 *    (2), DESMOE_ENCCL (3). desmoe_last_error() returns the message of the last
 *    failure on the calling thread.
 *  - Data-dependent checks the reference performs on the logits (finiteness,
 *    core.cpp:81-96) run on the device and latch a flag in the context; read it
 *    with desmoe_check(), which synchronises `stream`.
 *  - Expert-index outputs follow the reference's layout: per token the
 *    selected experts in ascending order (core.hpp:63-68), padded with -1 up
 *    to top_k; gates aligned, padded with 0.
 *  - All routing arithmetic is fp64 in the reference's operation order
 *    (SPEC.md:61); ties break to the lowest index everywhere.
 */
#ifndef DESMOE_H_
#define DESMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DESMOE_OK 0
#define DESMOE_EINVAL 1
#define DESMOE_ECUDA 2
#define DESMOE_ENCCL 3

/* GateActivation (core.hpp:11) plus IDENTITY: the input already holds gate
 * weights (topk_route(const GateMatrix&), gating.hpp:43). */
#define DESMOE_SOFTMAX 0
#define DESMOE_SIGMOID 1
#define DESMOE_IDENTITY 2

/* DesStrategy (des.hpp:16) plus VANILLA = plain top-K routing (gating.cpp:84) */
#define DESMOE_VANILLA (-1)
#define DESMOE_SEQ 0
#define DESMOE_VOTE 1

/* VoteSource (des.hpp:20) */
#define DESMOE_VOTE_ACTIVATED 0
#define DESMOE_VOTE_RAW_LOGITS 1

/* expert FFN kinds: the reference's synthetic linear D x D map
 * (ExpertBank, gating.hpp:48-63) and the north-star SwiGLU expert */
#define DESMOE_FFN_SWIGLU 0
#define DESMOE_FFN_LINEAR 1

typedef struct desmoe_ctx desmoe_ctx;
typedef struct desmoe_experts desmoe_experts;

/* Routing configuration = PoolConfig (core.hpp:13-19) + DesParams (des.hpp:20-24). */
typedef struct {
  int experts;      /* M = experts_total */
  int top_k;        /* K */
  int activation;   /* DESMOE_SOFTMAX | DESMOE_SIGMOID | DESMOE_IDENTITY */
  int strategy;     /* DESMOE_VANILLA | DESMOE_SEQ | DESMOE_VOTE */
  int seq_k;        /* DesParams::seq_k, strategy == SEQ */
  double vote_beta; /* DesParams::vote_beta, strategy == VOTE */
  int vote_source;  /* DESMOE_VOTE_ACTIVATED | DESMOE_VOTE_RAW_LOGITS */
} desmoe_route_cfg;

/* Device outputs of a routing call. Any pointer may be NULL if not wanted,
 * except route_* for the routing entry points. */
typedef struct {
  int* route_idx_dev;     /* [n x top_k] ascending experts, -1 padded        */
  double* route_gate_dev; /* [n x top_k] renormalised gates, 0 padded        */
  int* route_cnt_dev;     /* [n] = min(top_k, |coreset|)                    */
  int* coreset_dev;       /* [experts] ascending members (Coreset::members)  */
  int* coreset_size_dev;  /* [1]                                             */
  double* votes_dev;      /* [experts] VoteVector::votes (VOTE only)         */
  double* probs_dev;      /* [n x experts] activated gates (GateMatrix)      */
} desmoe_route_out;

/* ---- context --------------------------------------------------------------
 * One context per (device, host thread); owns workspaces, tensor maps and
 * CUDA graphs. Capacities bound every later call. */
int desmoe_create(desmoe_ctx** out, int device, int max_tokens, int max_experts,
                  int max_top_k, int max_hidden);
void desmoe_destroy(desmoe_ctx* ctx);
const char* desmoe_last_error(void);
/* Synchronises `stream` and reports (then clears) the device-side data
 * checks latched since the last call ("non-finite logit"). */
int desmoe_check(desmoe_ctx* ctx, void* stream);
int desmoe_version(void);

/* ---- validation (host only) ----------------------------------------------- */
/* validate_config (core.cpp:11-28): same invariants, same messages. */
int desmoe_validate_pool(int experts, int top_k, uint64_t bytes_per_expert, int hidden_dim);
/* vote_budget (des.cpp:29-31): floor(beta * experts). */
int desmoe_vote_budget(double beta, int experts);

/* validate_params (des.cpp:10-27): validate_config first, then the strategy's
 * parameter; same order, same messages. Host only. */
int desmoe_validate_params(const desmoe_route_cfg* cfg);

/* ---- gating / routing (logits in, device pointers) ------------------------
 * logits_dev is [n x experts] row-major, fp64 (the reference's RouterBlock,
 * core.hpp:32-44) or fp32 (the router GEMM's output / MOET trace values). */

/* activate (gating.cpp:10-40) -> probs [n x experts] fp64 */
int desmoe_activate(desmoe_ctx* ctx, const double* logits_dev, int n, int experts,
                    int activation, double* probs_dev, void* stream);

/* Full routing stage in one call:
 *   VANILLA: topk_route(activate(block), K)                (gating.cpp:84-97)
 *   SEQ/VOTE: des_run(block, cfg, params)                  (des.cpp:120-127)
 * also exposes the stage-1 products: coreset (for VANILLA the union of the
 * selections = unique_experts, gating.cpp:159-165) and votes. */
int desmoe_route(desmoe_ctx* ctx, const double* logits_dev, int n, const desmoe_route_cfg* cfg,
                 const desmoe_route_out* out, void* stream);
int desmoe_route_f32(desmoe_ctx* ctx, const float* logits_dev, int n,
                     const desmoe_route_cfg* cfg, const desmoe_route_out* out, void* stream);

/* ---- comparison policies (baselines.hpp / baselines.cpp) -------------------
 * BaselineParams (baselines.hpp:17-24). */
#define DESMOE_BASE_TOPK_REDUCE 0
#define DESMOE_BASE_NAEE 1
#define DESMOE_BASE_MCMOE 2
#define DESMOE_SCORE_MAX_GATE 0
#define DESMOE_SCORE_NEG_ENTROPY 1
typedef struct {
  int method;                      /* DESMOE_BASE_*                          */
  int k_reduced;                   /* TOPK_REDUCE: k in [1, top_k]           */
  double naee_beta;                /* NAEE: (0, 1)                           */
  double mcmoe_beta;               /* MCMOE: (0, 1)                          */
  double mcmoe_important_fraction; /* MCMOE: [0, 1]                          */
  int mcmoe_score;                 /* DESMOE_SCORE_*                         */
} desmoe_baseline_cfg;

/* baseline_route (baselines.cpp:125-137): topk_reduce_route (:10-16),
 * naee_route (:64-76) or mcmoe_route (:78-123) of logits_dev [n x experts]
 * (fp64; _f32 for router / trace logits). Writes route_idx/gate/cnt of `out`
 * (row stride top_k; NAEE / MC-MoE rows keep fewer than top_k, -1 / 0
 * padded) and, if given, probs_dev. Parameter errors carry the reference's
 * messages ("k_reduced outside [1, top_k]", "naee beta outside (0, 1)",
 * "mcmoe beta outside (0, 1)", "important_fraction outside [0, 1]");
 * non-finite logits are reported by desmoe_check. */
int desmoe_baseline_route(desmoe_ctx* ctx, const double* logits_dev, int n,
                          const desmoe_route_cfg* cfg, const desmoe_baseline_cfg* params,
                          const desmoe_route_out* out, void* stream);
int desmoe_baseline_route_f32(desmoe_ctx* ctx, const float* logits_dev, int n,
                              const desmoe_route_cfg* cfg, const desmoe_baseline_cfg* params,
                              const desmoe_route_out* out, void* stream);

/* ---- MOET router traces (trace.hpp:30-85, trace.cpp:122-442) ----------------
 * The reference's trace file format, so captured router traces feed the
 * routing entry points in logits-in mode. Binary v1: "MOET", u16 version,
 * u8 model, u8 reserved, u32 experts/top_k/layers/block_size/steps, u64 seed,
 * f32 rho/temperature, then per (step, layer) record u32 step, u32 layer and
 * block_size x experts f32 logits, little-endian. JSONL: a header object line
 * and one {"layer","logits","step"} line per record. Host-only (no GPU). */
#define DESMOE_MOET_BINARY 0
#define DESMOE_MOET_JSONL 1
/* TraceError::Code (trace.hpp:58-66) */
#define DESMOE_MOET_IO 0
#define DESMOE_MOET_BAD_MAGIC 1
#define DESMOE_MOET_BAD_VERSION 2
#define DESMOE_MOET_BAD_HEADER 3
#define DESMOE_MOET_TRUNCATED 4
#define DESMOE_MOET_SHAPE_MISMATCH 5
#define DESMOE_MOET_BAD_VALUE 6

typedef struct { /* TraceHeader (trace.hpp:30-40) */
  int experts, top_k, layers, block_size, steps;
  int model; /* SynthModel: 0 iid_gaussian, 1 dirichlet, 2 shared_bias */
  double rho, temperature;
  uint64_t seed;
} desmoe_moet_header;

/* decode_trace (trace.cpp:432-441; format sniffed from the first byte).
 * `logits` (may be NULL: validate and read the header only) receives
 * steps*layers*block_size*experts doubles in (step, layer) record order.
 * Errors: DESMOE_EINVAL, the reference's message in desmoe_last_error() and
 * the TraceError code in *trace_code. */
int desmoe_moet_decode(const void* bytes, size_t len, desmoe_moet_header* header,
                       double* logits, int* trace_code);
/* encode_trace (trace.cpp:422-430): out == NULL -> *len = bytes needed. */
int desmoe_moet_encode(const desmoe_moet_header* header, const double* logits, int format,
                       void* out, size_t* len, int* trace_code);

/* Stage 1 only: des_seq_coreset (des.cpp:33-45) / des_vote_coreset
 * (des.cpp:65-95, also the contract of fused_vote_pipeline des.cpp:166-224).
 * cfg->strategy selects which; out->coreset_dev / coreset_size_dev required. */
int desmoe_coreset(desmoe_ctx* ctx, const double* logits_dev, int n,
                   const desmoe_route_cfg* cfg, const desmoe_route_out* out, void* stream);

/* Stage 2 only: constrained_route (des.cpp:97-118) over a caller-given
 * coreset (ascending, unique, host array of n_members entries). */
int desmoe_constrained_route(desmoe_ctx* ctx, const double* logits_dev, int n,
                             const desmoe_route_cfg* cfg, const int* members_host,
                             int n_members, const desmoe_route_out* out, void* stream);

/* select_top_gates (gating.cpp:42-71), both overloads, any k <= candidates:
 * the k largest of values_dev[0..m) by (value desc, index asc), restricted to
 * cand_dev[0..n_cand) when cand_dev != NULL (ascending, unique, < m); writes
 * the k selected indices in ascending order to out_dev. m <= 16384. */
int desmoe_select_top(desmoe_ctx* ctx, const double* values_dev, int m, int k,
                      const int* cand_dev, int n_cand, int* out_dev, void* stream);

/* renormalize_over (gating.cpp:73-82): out[j] = values[sel[j]] / sum, the
 * sum taken over sel in the given order. */
int desmoe_renormalize(desmoe_ctx* ctx, const double* values_dev, const int* sel_dev, int count,
                       double* out_dev, void* stream);

/* ---- permutation (K3) -------------------------------------------------------
 * Per-expert counts (moe_latency's count route, analysis.cpp:16-30), ascending
 * exclusive offsets, stable (ascending token) slot lists, the ascending list of
 * active experts (unique_experts, gating.cpp:159-165) and its size U. */
int desmoe_permute(desmoe_ctx* ctx, const int* route_idx_dev, const int* route_cnt_dev, int n,
                   int top_k, int experts, int* expert_count_dev, int* expert_offset_dev,
                   int* slot_of_dev, int* slot_token_dev, int* active_dev, int* n_active_dev,
                   void* stream);

/* ---- experts (K4) -----------------------------------------------------------
 * Registers device-resident bf16 expert weights: they are packed once into a
 * context-owned tile-contiguous copy the FFN kernel streams (the caller's
 * tensors are only read during this call; synchronises). SWIGLU: w_gate/w_up [experts x ffn x hidden], w_down
 * [experts x hidden x ffn]. LINEAR: w_gate = W [experts x hidden x hidden]
 * (ExpertBank::expert_weights layout [out][in], gating.cpp:122-134),
 * w_up = w_down = NULL, ffn = hidden. hidden % 128 == 0, ffn % 128 == 0. */
int desmoe_experts_create(desmoe_ctx* ctx, int kind, int experts, int hidden, int ffn,
                          const void* w_gate_dev, const void* w_up_dev, const void* w_down_dev,
                          desmoe_experts** out);
void desmoe_experts_destroy(desmoe_experts* ex);

/* ---- expert parallelism (EP) -------------------------------------------------
 * A world of up to 8 ranks (one process per GPU of an NVSwitch box) shards
 * the experts in contiguous ranges, rank r owning [expert_lo, expert_hi).
 * Router, coreset and re-route are replicated (deterministic, so every rank
 * derives the identical route with no exchange). Each rank streams only its
 * experts; its FFN epilogues push every gate-scaled slot row straight into
 * all ranks' slot buffers over NVLink peer memory and signal each rank's
 * arrival counter; each rank's combine waits for all arrivals and sums the
 * slots in ascending expert order — bit-identical to one GPU.
 *
 * desmoe_experts_create_ep: like desmoe_experts_create, but the weight
 * pointers hold only the owned experts (expert_hi - expert_lo of them) while
 * `experts` is the pool size M the router sees. */
int desmoe_experts_create_ep(desmoe_ctx* ctx, int kind, int experts, int expert_lo, int expert_hi,
                             int hidden, int ffn, const void* w_gate_dev, const void* w_up_dev,
                             const void* w_down_dev, desmoe_experts** out);
/* The exchange buffers this rank exposes (each the base of its own
 * cudaMalloc, ready for cudaIpcGetMemHandle): the two-epoch slot buffer and
 * the arrival counter. Allocates on first call; synchronises. */
int desmoe_ep_local_buffers(desmoe_experts* ex, void** slot_buf, size_t* slot_bytes,
                            void** flag_buf, size_t* flag_bytes);
/* peer_*[r] = rank r's buffers as mapped in this process (cudaIpcOpenMemHandle;
 * entry `rank` = this rank's own local buffers). world == 1 disconnects. Every
 * rank must then call desmoe_layer_forward the same number of times with the
 * same route configuration (the exchange is per call). */
int desmoe_ep_connect(desmoe_experts* ex, int world, int rank, void* const* peer_slot_bufs,
                      void* const* peer_flag_bufs);

/* Cross-process wiring: desmoe_ep_export writes this rank's 128-byte handle
 * (CUDA IPC handles of its slot buffer and arrival counter); the caller
 * all-gathers the handles in rank order (any transport: torch.distributed,
 * MPI, a file) and passes them to desmoe_ep_import, which maps the peers'
 * buffers (NVLink peer memory) and connects. */
#define DESMOE_EP_HANDLE_BYTES 128
int desmoe_ep_export(desmoe_experts* ex, void* handle_out);
int desmoe_ep_import(desmoe_experts* ex, int world, int rank, const void* handles);

/* Expert FFN + combine for a routed block (moe_forward, gating.cpp:136-157):
 * y[t] = sum over the token's experts in ascending order of gate * expert(x_t).
 * x_dev [n x hidden] bf16, route_* as produced by desmoe_route, y_dev
 * [n x hidden] fp32. Streams each active expert's weights once. */
int desmoe_expert_ffn(desmoe_ctx* ctx, const desmoe_experts* ex, const void* x_dev, int n,
                      int top_k, const int* route_idx_dev, const double* route_gate_dev,
                      const int* route_cnt_dev, float* y_dev, void* stream);

/* moe_forward (gating.cpp:136-157) over the reference's linear experts in
 * fp64, bit-identical to the CPU library (same operation order, no FMA
 * contraction): y[t] = sum over the token's experts in stored order of
 * gate * W_e x_t. w_dev [experts x hidden x hidden] ([out][in], the
 * ExpertBank layout), x_dev [n x hidden], y_dev [n x hidden], route_* as
 * desmoe_route writes them (row stride top_k). Expert indices must lie in
 * [0, experts) (the caller validates, as moe_forward does). */
int desmoe_moe_forward_f64(desmoe_ctx* ctx, const double* w_dev, const double* x_dev, int n,
                           int hidden, int experts, int top_k, const int* route_idx_dev,
                           const double* route_gate_dev, const int* route_cnt_dev, double* y_dev,
                           void* stream);

/* ---- router GEMM (K1) -------------------------------------------------------
 * logits[n x experts] fp32 = x[n x hidden] (bf16) . w_router[experts x hidden]^T
 * (bf16). The reference takes logits as input; this is the producer the
 * paper's layer puts in front of it. */
int desmoe_router_logits(desmoe_ctx* ctx, const void* x_dev, const void* w_router_dev, int n,
                         int experts, int hidden, float* logits_dev, void* stream);

/* ---- whole layer --------------------------------------------------------------
 * router -> activation/top-K -> coreset -> constrained route -> permute ->
 * expert FFN + combine. stats_dev (optional, int[4]): {U unique experts,
 * coreset size, total selections, experts streamed by this rank (= U unless
 * expert-parallel)}. */
int desmoe_layer_forward(desmoe_ctx* ctx, const desmoe_experts* ex, const void* w_router_dev,
                         const void* x_dev, int n, const desmoe_route_cfg* cfg, float* y_dev,
                         int* stats_dev, void* stream);

/* A stack of `layers` DES MoE layers applied in sequence to one block (the
 * MoE layers of one diffusion denoising step): x_dev [n x hidden] bf16 ->
 * y_dev [n x hidden] fp32; layer l's output feeds layer l+1 as bf16 through
 * context-owned buffers. The whole stack is captured into ONE CUDA graph
 * (re-captured when any argument changes). stats_dev: optional int[4*layers].
 * residual != 0: each layer outputs h + MoE(h) (the residual stream a model's
 * MoE blocks sit on), so token diversity survives the stack. */
int desmoe_stack_forward(desmoe_ctx* ctx, desmoe_experts* const* experts,
                         const void* const* w_router_dev, int layers, const void* x_dev, int n,
                         const desmoe_route_cfg* cfg, float* y_dev, int* stats_dev, int residual,
                         void* stream);

/* The fp32 router logits [n x experts] the last desmoe_layer_forward on this
 * context routed with (for checking its routing against the reference). */
int desmoe_layer_logits(desmoe_ctx* ctx, float* logits_dev, int n, int experts, void* stream);

/* The route of the last desmoe_layer_forward on this context (layout of
 * desmoe_route_out; any pointer may be NULL): route_idx/gate [n x top_k],
 * route_cnt [n], coreset members [experts] + count (DES strategies). */
int desmoe_layer_route(desmoe_ctx* ctx, int* route_idx_dev, double* route_gate_dev,
                       int* route_cnt_dev, int* members_dev, int* n_members_dev, int n, int top_k,
                       int experts, void* stream);

/* Same with HOST buffers: copies x (bf16) in, runs the layer, copies y
 * (fp32) and stats back; synchronises. The end-to-end entry a C/C++ caller
 * without device memory uses. */
int desmoe_layer_forward_host(desmoe_ctx* ctx, const desmoe_experts* ex,
                              const void* w_router_dev, const void* x_host, int n,
                              const desmoe_route_cfg* cfg, float* y_host, int* stats_host,
                              void* stream);

/* desmoe_layer_forward captures its launch sequence into a CUDA graph the
 * first time it sees a given (experts, router, x, n, cfg, y, stats) tuple and
 * replays it afterwards; enable = 0 launches eagerly instead. Default on. */
int desmoe_set_graphs(desmoe_ctx* ctx, int enable);

/* ---- live phase timing -------------------------------------------------------
 * When enabled, desmoe_layer_forward records CUDA events on its stream between
 * its phases: [0] router GEMM + gating + coreset + constrained re-route (one
 * cluster kernel; split into [0] router GEMM, [1] routing kernels for shapes
 * outside its envelope), then the persistent expert FFN (permutation, gather,
 * gate/up + down GEMMs), [last] (expert-parallel arrival wait +) ordered
 * combine. desmoe_get_phase_ms synchronises on the last event and writes up
 * to max_phases elapsed times (ms) of the LAST call; returns the number
 * written, or minus a DESMOE_E* code on failure. */
int desmoe_set_profiling(desmoe_ctx* ctx, int enable);
int desmoe_get_phase_ms(desmoe_ctx* ctx, float* ms_out, int max_phases);
/* Kernels launched by the last desmoe_layer_forward call. */
int desmoe_last_launch_count(desmoe_ctx* ctx);
/* Timeline tracing of the persistent expert-FFN kernel (profiling aid):
 * buf_dev[0] is an append cursor (zero it before a call), followed by
 * `capacity` records of two u64 {unit<<32 | cta<<8 | event, globaltimer ns};
 * events 0 start, 1 gather done, 2 unit dequeued, 3 unit epilogue done,
 * 5 CTA exit, 6 activations ready, 7 H ready. capacity 0 disables. Takes
 * effect on the next (re)captured launch sequence. */
int desmoe_set_trace(desmoe_ctx* ctx, uint64_t* buf_dev, int capacity);

#ifdef __cplusplus
}
#endif

#endif /* DESMOE_H_ */

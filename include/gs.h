/* gs.h — C-ABI of the GenServe DiT-step hot path on B200 (libgs.so).
 *
 * The calls follow the paper's statement of the scheduling problem (§4.4,
 * P:408-420): a request r is allocated a GPU set X_r(t) with |X_r| in {0} u P,
 * P = {1, 2, 4, 8} (P:92 Listing genserve-api, "elastic_sp=[1,2,4,8]"; "Images use
 * at most one GPU ... videos use |X_v(t)| in {0} u P"), and the transition
 * X_r(t) -> X_r(t + D_round) expresses start, continue, preempt, resume and reconfigure
 * (P:415).  Preemption happens only at denoising-step boundaries and the latent stays in
 * device memory (§1; §4.2 "its latent state is retained in device memory");
 * SP degree changes between steps (§4.3, "downgrading the SP degree").
 * One "step" is one reverse-diffusion step (P:129-133 Eq. reverse) = one DiT forward + a
 * FlowMatch-Euler update (DESIGN.md readings).
 *
 * Ranks and processes.  A context owns one CUDA device and one or more *ranks* (global
 * indices into the job's GPUs).  Production: one process per GPU (torchrun), each with one
 * rank; SP exchanges use NCCL over NVLink (gs_init with an NCCL unique id).  Test fixture:
 * gs_init_emulated() puts W virtual ranks in one process on one device and performs the
 * same exchanges with device copies (all calls then act on every rank at once).
 * All calls that move data between ranks (gs_submit, gs_run_steps, gs_resume) are
 * collective over the ranks they name: every process owning one of those ranks must make
 * the same call with the same arguments (SPMD).
 *
 * Errors.  Every call returns GS_OK (0) or a negative GS_E* code; nothing throws across the
 * ABI.  gs_last_error() returns a context-owned message valid until the next call on that
 * context.  Pointers: "host" arguments are borrowed for the duration of the call; "device"
 * arguments (debug entry points only) must be device memory of the context's device, owned
 * by the caller.  The context owns all memory it allocates (weights, latents, arenas).
 */
#ifndef GS_H_
#define GS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gs_ctx gs_ctx;
typedef uint64_t gs_req;
typedef uint64_t gs_ticket; /* an asynchronous run (gs_run_steps_async / gs_wait) */

enum {
  GS_OK = 0,
  GS_EINVAL = -1,        /* bad shape / argument ("UnknownConfiguration")        */
  GS_ESTATE = -2,        /* contract violation: wrong placement, paused, overlap    */
  GS_ENOMEM = -3,        /* device allocation failed                                        */
  GS_ECUDA = -4,         /* CUDA runtime / kernel error                                     */
  GS_ENCCL = -5,         /* NCCL error                                                      */
  GS_EUNSUPPORTED = -6   /* configuration not supported by this build                       */
};

/* Request states.  QUEUED: submitted, holds no GPU (|X_r| = 0) until gs_place; PLACED: its
 * latent is sharded on a GPU set and it may run; RUNNING: inside a run; PAUSED: preempted at a step
 * boundary, latent kept in device memory (§4.2) until gs_resume; DONE: all steps run. */
enum { GS_REQ_PLACED = 0, GS_REQ_RUNNING = 1, GS_REQ_PAUSED = 2, GS_REQ_DONE = 3, GS_REQ_QUEUED = 4 };

/* DiT model shape (SURVEY.md §8 shape table; Wan2.1-style block, reading 1).
 * Weights are generated on the device from the counter RNG:
 * block l uses seed weight_seed + l, global tensors weight_seed + 1000000. */
typedef struct {
  int dim;        /* D, multiple of 64, <= 8192                        */
  int heads;      /* H, head dim D/H in {64, 128}                      */
  int ffn;        /* F, multiple of 256                                */
  int layers;     /* L                                                 */
  int lat;        /* latent floats per token (64)                      */
  int freq_dim;   /* sinusoidal time-embedding width (256)            */
  float rope_theta; /* 10000                                           */
  float eps;      /* LayerNorm / RMSNorm epsilon (1e-6)                */
  float flow_shift; /* FlowMatch shift s (5.0)                         */
  uint64_t weight_seed;
  /* Text cross-attention in every block (the paper's DiT blocks "perform N
   * denoising steps with cross-attention for text alignment", §2.1; Wan2.1 layout, DESIGN.md
   * reading 19).  0 = the north-star block (self-attention + MLP only). */
  int cross_attn;
  int text_len;   /* context tokens (512)                                */
  int text_dim;   /* prompt-embedding width (4096), multiple of 64       */
} gs_model_desc;

/* ------------------------------------------------------------------ context */
/* Writes NCCL's 128-byte unique id to out (host, >= 128 bytes). Call on one process and
 * broadcast the bytes (e.g. with torch.distributed) before gs_init. */
int gs_nccl_unique_id(void* out128);
/* One process per GPU: `device` is the local CUDA ordinal, `rank` in [0, world_size).
 * world_size == 1 needs no unique id (nccl_uid may be NULL). */
int gs_init(int device, int world_size, int rank, const void* nccl_uid, gs_ctx** out);
/* Test fixture: world_size virtual ranks on one device in this process (exchanges are
 * device-to-device copies; same kernels and shard shapes as the NCCL path). */
int gs_init_emulated(int device, int world_size, gs_ctx** out);
void gs_destroy(gs_ctx* ctx);
const char* gs_last_error(gs_ctx* ctx);
/* Runtime options.  "a2a": 1 (default) = fused all-to-alls by peer stores wherever the SP degree
 * divides the heads (the QKV pack kernel and the attention epilogue store straight into the
 * consuming GPU's buffers over NVLink -- CUDA IPC mappings exchanged over NCCL at gs_run_steps
 * -- ordered by a flag barrier), 0 = transfer plans (grouped ncclSend/Recv, or
 * device copies in emulated mode).  Both give bit-identical results.  Every process of an SP
 * group must use the same setting.  "gemm_bn": GEMM pair-tile width, 0 (default: 256, or 192 when
 * N % 192 == 0 and the narrower tiles fill a small grid's last wave better), 192 or 256 forced
 * (process-wide; both give identical bits).  "pdl": 1 (default) launches the step's kernels with
 * programmatic dependent launch (each kernel's setup overlaps the previous kernel's drain), 0 plain
 * stream order (process-wide; identical bits).  "usp_ring": 1 (default) Ulysses only; 2, 4 or 8 = the USP hybrid's ring
 * degree for batches whose p it divides with p / ring dividing the heads (gs_plan_a2a_usp; identical
 * bits; every process of an SP group must use the same value).  GS_EINVAL for an unknown key or value. */
int gs_set_option(gs_ctx* ctx, const char* key, long long value);
/* Number of SMs of the context's device, world size, ranks owned by this process. */
int gs_info(gs_ctx* ctx, int* num_sms, int* world_size, int* nlocal);

/* ------------------------------------------------------------------ models */
int gs_model_create(gs_ctx* ctx, const gs_model_desc* desc, int* model_id);
/* Copy one weight tensor to host (parity rung T1). layer = -1 for global tensors.
 * name in {w_qkv,b_qkv,g_q,g_k,w_o,b_o,w_1,b_1,w_2,b_2,mod} (block) or
 * {w_pe,b_pe,w_t1,b_t1,w_t2,b_t2,w_tp,b_tp,mod_head,w_head,b_head} (global); cross-attention
 * models add {ln3_w,ln3_b,w_cq,b_cq,w_ckv,b_ckv,g_cq,g_ck,w_co,b_co} and {w_te1,b_te1,w_te2,b_te2}.
 * bytes must equal the tensor size (bf16 tensors: 2 B/elem, mod tables fp32). */
int gs_get_weight(gs_ctx* ctx, int model, int layer, const char* name, void* host, size_t bytes);

/* ------------------------------------------------------------------ requests */
/* Submit a request: "submit a request's resolution, frames and steps" (BASELINE.json north_star);
 * a request is a fixed number of reverse-diffusion steps (§2.1 Eq. reverse).  Resolution
 * w x h (multiples of 16), frames (1 for images, = 1 mod 4), `steps` denoising steps (sigma
 * schedule of DESIGN.md reading 5).  The initial latent z_T [n, lat] fp32 (token-major,
 * n = (1 + (frames-1)/4) * (h/16) * (w/16)) is generated from noise_seed, or copied from
 * init_latent (host, exactly n*lat floats, borrowed for the call) if non-NULL.
 * Placement: with ranks != NULL the request is placed at once, token-sharded on `ranks`
 * (p = nranks in {1,2,4,8}, distinct, in SP order; = gs_submit + gs_place).  With ranks == NULL and
 * nranks == 0 it is QUEUED: it holds no GPU until gs_place (the scheduler's start action).
 * Multi-process (NCCL) contexts: gs_submit is collective over the WHOLE job (every process submits
 * every request, so request ids agree job-wide and any process can later receive a shard on
 * resume; checked with one all-reduce, GS_ESTATE on a mismatch).  Errors: GS_EINVAL bad shape /
 * ranks, GS_ENOMEM, GS_ECUDA. */
int gs_submit(gs_ctx* ctx, int model, int width, int height, int frames, int steps,
              uint64_t noise_seed, const float* init_latent, const int* ranks, int nranks,
              gs_req* out);
/* Submit a request of a cross-attention model with its prompt (P:759 / Tab. paused_memory: the
 * VideoState keeps the prompt embeddings).  cfg_scale > 0 runs classifier-free guidance with
 * guidance g = cfg_scale (a cond and an uncond branch per step, v = v_u + g (v_c - v_u), DESIGN.md
 * reading 21); cfg_scale <= 0 runs the cond branch only.  prompt_embeds: host bf16
 * [nb][text_len][text_dim] (nb = 2 with CFG: cond, then uncond; exactly that many elements are
 * read), or NULL for the synthetic prompt of prompt_seed.  Other
 * arguments as gs_submit. */
int gs_submit_text(gs_ctx* ctx, int model, int width, int height, int frames, int steps,
                   uint64_t noise_seed, uint64_t prompt_seed, float cfg_scale,
                   const float* init_latent, const void* prompt_embeds, const int* ranks,
                   int nranks, gs_req* out);
/* First placement of a QUEUED request on `ranks` (the "start" action of X_r(t): |X_r| goes from 0
 * to p, §4.4; images on one GPU, videos on p in {1,2,4,8}): allocates the latent
 * shards and writes z_T.  Collective over the processes owning `ranks`.  GS_ESTATE if the request
 * is not QUEUED or a rank belongs to an in-flight run; GS_EINVAL bad ranks. */
int gs_place(gs_ctx* ctx, gs_req req, const int* ranks, int nranks);
/* Run k steps of a batch of requests: the "start / continue" actions for one scheduling round
 * (§4.4); one step = one DiT forward + Euler update (§2.1).  Preconditions
 * (GS_ESTATE otherwise): every request is PLACED on exactly `ranks`, all use the same model, no
 * rank belongs to another in-flight run (capacity / no-overlap rule, Eq. capacity, Alg.1
 * P:498), and in multi-process mode this process owns one of `ranks`; k <= remaining steps of each
 * (GS_EINVAL).  Returns after the last step, or after the step boundary at which a preemption was
 * requested (§1: preemption only at step boundaries); steps actually run -> *steps_run.
 * Bit-exact w.r.t. SP degree, batch composition and preempt/resume.
 * = gs_run_steps_async + gs_wait. */
int gs_run_steps(gs_ctx* ctx, const gs_req* reqs, int nreq, const int* ranks, int nranks, int k,
                 int* steps_run);
/* Asynchronous gs_run_steps: validates and claims the GPU set, then runs the k steps on a worker
 * thread of the context (on the stream of ranks[0]) and returns at once with a ticket.  Runs on
 * disjoint GPU sets proceed concurrently ("each GPU either processes one batch or is idle",
 * P:390-398 §4.3; disjoint SP groups).  Validation errors are returned here (no ticket);
 * errors of the run itself are returned by gs_wait.  Every ticket must be waited for. */
int gs_run_steps_async(gs_ctx* ctx, const gs_req* reqs, int nreq, const int* ranks, int nranks,
                       int k, gs_ticket* ticket);
/* Wait for a run: returns its status (first error of the run, message in gs_last_error) and the
 * steps it ran (steps_run may be NULL); releases its GPU set.  GS_EINVAL for an unknown ticket. */
int gs_wait(gs_ctx* ctx, gs_ticket ticket, int* steps_run);
/* 1 if the run has finished (gs_wait will not block), 0 if it is still running, GS_EINVAL for
 * an unknown ticket. */
int gs_ticket_done(gs_ctx* ctx, gs_ticket ticket);
/* Request preemption (pause): "preempting ... at step boundaries; its latent state is retained
 * in device memory" (§1; §4.2; "a pause requested mid-step takes effect at
 * the current step's completion").  If the request is in a run, the run stops after its current
 * step; otherwise it is paused at once.  Thread-safe (any thread, while runs are in flight).
 * GS_ESTATE for a DONE request.  steps_done_out (may be NULL) = steps completed so far. */
int gs_preempt(gs_ctx* ctx, gs_req req, int* steps_done_out);
/* Resume / reconfigure at a step boundary onto `ranks` (p' = nranks): "resume ... possibly at a
 * different SP degree" (§4.2, §4.3 runtime SP degree switching; reconfigure
 * when the request was not paused).  Re-shards the latent (pure copy of contiguous token
 * ranges, interval intersections of old and new shards).  Collective over
 * the processes owning old or new ranks.  GS_ESTATE if the request is RUNNING / DONE / QUEUED or a
 * new rank belongs to an in-flight run (multi-process contexts: an old rank too, since the re-shard
 * is collective over its process). */
int gs_resume(gs_ctx* ctx, gs_req req, const int* ranks, int nranks);
/* state in GS_REQ_*; ranks_out (host, >= 8 ints) may be NULL. */
int gs_query(gs_ctx* ctx, gs_req req, int* steps_done, int* steps_total, int* nranks,
             int* ranks_out, int* state, int* n_tokens);
/* Copy the latent [n, lat] fp32 to host (nfloats must equal n*lat): every shard owned by this
 * process is written to its token range (in emulated mode: the whole latent).  GS_ESTATE while the
 * request is RUNNING or QUEUED. */
int gs_read_latent(gs_ctx* ctx, gs_req req, float* host, size_t nfloats);
/* Free a request's device state (GS_ESTATE while RUNNING). */
int gs_release(gs_ctx* ctx, gs_req req);

/* ------------------------------------------------------------------ VAE decode (NEXT-4)
 * The pipeline stage after the DiT: "a VAE for latent encoding/decoding" (§2.1), decoupled
 * from the DiT and always run on a single GPU (§4.3; Tab. stage_breakdown).
 * Decoder shape: Wan2.1-VAE-like causal 3-D conv decoder (DESIGN.md §NEXT-4 readings V1-V8; the
 * module walk of synth/vae.py): de-normalise + unpatchify the DiT latent, 1x1x1 conv, conv_in,
 * residual blocks, temporal (x2, first-frame rule) and spatial (x2 nearest + conv) upsampling,
 * RMS norm + SiLU + conv_out, clamp to [-1, 1].  Weights are generated on the device from the
 * counter RNG (tensor id 200 + 4 * module + slot, seed weight_seed). */
typedef struct {
  int z_dim;          /* latent channels (16)                                            */
  int dims[5];        /* decoder widths (384, 384, 384, 192, 96)                          */
  int blocks;         /* residual blocks per up stage (3)                                 */
  int mid_blocks;     /* residual blocks at the latent resolution (2)                     */
  int temporal_up[3]; /* temporal x2 in up stages 0..2 (1, 1, 0)                          */
  int out_ch;         /* output channels (3)                                              */
  uint64_t weight_seed;
} gs_vae_desc;
int gs_vae_create(gs_ctx* ctx, const gs_vae_desc* desc, int* vae_id);
/* Decode one latent on local rank `rank` (a single GPU): latent [F * Ht * Wt, 64] fp32 in DiT token
 * layout (host, or device memory of the context's device when flags & 1), video
 * [T_out][16 Ht][16 Wt][out_ch] fp32 (host, or device when flags & 2), T_out = F after the temporal
 * stages (1 + 4 (F - 1) for the Wan shape).  Activation buffers are taken from and returned to the
 * context's pool.  GS_EINVAL bad shape; GS_ENOMEM; GS_ECUDA. */
int gs_vae_decode(gs_ctx* ctx, int vae_id, int rank, const float* latent, int F, int Ht, int Wt, float* video,
                  int flags);
/* Decode a request's latent (the stage after its last DiT step) on ONE of its GPUs: the latent is
 * gathered from its shards onto ranks[0] of the request (emulated contexts; multi-process
 * contexts need the whole request on this process).  video: host fp32 as gs_vae_decode. */
int gs_vae_decode_request(gs_ctx* ctx, int vae_id, gs_req req, float* video);
/* Parity entry point: one causal 3-D convolution (oracle/vae.py causal_conv3d) on device buffers,
 * x bf16 [T][H][W][Cp], w bf16 [Coutp][kt][kh][kw][Cp], bias bf16 [Coutp], resid bf16
 * [T][H][W][Coutp] or NULL, out per mode (0 bf16 [T][H][W][out_cs]; 1 temporal interleave;
 * 2 fp32 clamp [T][H][W][out_real]). */
int gs_debug_conv3d(gs_ctx* ctx, const void* x, const void* w, const void* bias, const void* resid, void* out,
                    int T, int H, int W, int Cp, int kt, int kh, int kw, int Coutp, int out_cs, int mode,
                    int out_real);

/* ------------------------------------------------------------------ measurement */
/* enable = 1: per-kernel-class and per-step CUDA-event timing inside gs_run_steps (events on the
 * launching stream); 2: per-step events only (two per step, no per-kernel events); 0: off.
 * gs_stats writes a JSON object {"class": {"ms": total, "n": launches}, ...,
 * "step_ms": [device time of each profiled step], "a2a_peer": exchanges run as peer stores,
 * "a2a_plan": exchanges run as transfer plans,
 * "launches": total kernel launches} accumulated since the last reset (a2a counts: since init). */
int gs_profile(gs_ctx* ctx, int enable, int reset);
int gs_stats(gs_ctx* ctx, char* json, size_t len);
/* The CUDA stream (cudaStream_t) the context launches rank `rank`'s work on, as a pointer. */
int gs_stream(gs_ctx* ctx, int rank, void** stream_out);

/* ------------------------------------------------------------------ exchange plans (host only)
 * The SP data movement of one DiT block (Ulysses seq->head of
 * Q,K,V and head->seq of O) and of a resume (row a17: latent re-shard p -> p') as transfer lists
 * for one participant.  Pure host computation (no GPU, no context): the NCCL executor, the
 * emulated executor and the CPU multi-process tests all run these plans.  Messages between a
 * pair of participants are matched in list order (NCCL point-to-point semantics).
 * Offsets / sizes are in elements of the named buffers (bf16 for a2a, fp32 for the latent).
 * Head partition (reading 9): every position holds Hf = floor(H/p) full heads; the
 * R = H mod p remaining heads are cut into c = p / gcd(R, p) query chunks each ([ci n/c, (ci+1) n/c)
 * of every request), dealt out in order R / gcd(R, p) per position, so all positions do H/p heads
 * of attention work.  Token shard i of p is [floor(i n/p), floor((i+1) n/p)) (reading 10).
 *   SEND buffer of a position (pack-kernel layout): chunks j < p = [rows_me][Hf][d] (full heads of
 *     position j), then chunk p+u = [rows_me][d] (partial head Hf p + u);
 *   RECV buffer: full heads [rows of the whole batch][Hf][d], then per local unit t a K / V block
 *     [rows of the batch][d] (kind 0) or a Q block [chunk rows of every request][d] (kind 2);
 *   a2a kind 1 (O): O buffer in the kind-2 (Q) layout (attention output), STAGE buffer
 *     (*stage_elems elements), ORECV buffer [rows_me][heads * d]; COPY entries (2-D blocks) run
 *     after all sends/recvs completed;
 *   reshard: OLD shard [old rows][lat], NEW shard [new rows][lat]; peers are global ranks. */
enum { GS_XFER_SEND = 0, GS_XFER_RECV = 1, GS_XFER_COPY = 2 };
enum { GS_BUF_SEND = 0, GS_BUF_RECV = 1, GS_BUF_O = 2, GS_BUF_STAGE = 3, GS_BUF_ORECV = 4,
       GS_BUF_OLD = 5, GS_BUF_NEW = 6 };
typedef struct {
  int op;                  /* GS_XFER_*                                                    */
  int peer;                /* SP position (a2a) or global rank (reshard); -1 for COPY       */
  int src_buf, dst_buf;    /* GS_BUF_* (-1 where unused)                                   */
  long long src_off, dst_off;
  long long rows, width;   /* a rows x width block                                         */
  long long src_pitch, dst_pitch;
} gs_xfer;
/* kind 0 = seq->head of K and V, 2 = seq->head of Q, 1 = head->seq of O, for SP position `me` of p
 * over a batch of nreq requests with n_tokens[r] tokens.  out may be NULL to query *n_out; GS_EINVAL if max_out is
 * too small or an argument is out of range. */
int gs_plan_a2a(int kind, int p, int me, int nreq, const int* n_tokens, int heads, int head_dim,
                gs_xfer* out, int max_out, int* n_out, long long* stage_elems);
/* The same for the USP hybrid (NEXT-2; xFuser's Unified Sequence Parallelism, §5): p = u x ring,
 * every head cut into `ring` query chunks, unit (head h, chunk ci) on position (h / (H/u)) * ring + ci;
 * each unit receives its query chunk and the head's K / V of every token in token order (the ring's
 * K / V exchange as an in-order all-gather), so results are bit-exact with plain Ulysses.  Falls back
 * to gs_plan_a2a's partition when ring does not divide p or p / ring does not divide heads. */
int gs_plan_a2a_usp(int kind, int p, int ring, int me, int nreq, const int* n_tokens, int heads, int head_dim,
                    gs_xfer* out, int max_out, int* n_out, long long* stage_elems);
/* Peer-store addressing of the fused all-to-alls (p divides heads; DESIGN.md §8 "fused exchange"):
 * the QKV pack kernel of SP position `me` stores local row m of request r as full-batch row
 * m + row_delta[r] of the RECV buffer of the position owning each head, and its attention kernel
 * stores the output row of token t of request r into the owner i = max{i : own_lo[r*p+i] <= t} at
 * element o_base[r*p+i] + t*heads*head_dim + (h - me*heads/p)*head_dim of that owner's ORECV
 * buffer [rows_i][heads*head_dim].  Outputs: row_delta [nreq], own_lo [nreq*p], o_base [nreq*p].
 * GS_EUNSUPPORTED when p does not divide heads (those batches use the gs_plan_a2a transfers). */
int gs_plan_peer(int p, int me, int nreq, const int* n_tokens, int heads, int head_dim,
                 long long* row_delta, int* own_lo, long long* o_base);
/* Re-shard of a request's latent [n_tokens, lat] from old_ranks (old_p) to new_ranks (new_p), as
 * seen by global rank `me` (which may be in either set, both or none). */
int gs_plan_reshard(int n_tokens, int lat, const int* old_ranks, int old_p, const int* new_ranks,
                    int new_p, int me, gs_xfer* out, int max_out, int* n_out);

/* ------------------------------------------------------------------ parity / debug entry points
 * Single device, rank-independent, caller-owned buffers.  The launch is ordered after all work
 * previously submitted to the legacy default stream (where torch writes the caller's inputs)
 * and the call returns after the kernel completed. */
/* GEMM C = A W^T with epilogue epi (0 bf16, 1 GELU-bf16, 2 fp32, 3 gated-residual fp32,
 * 4 Euler fp32; see csrc/kernels.h).  A [M,K] bf16, W [N,K] bf16, bias [N] bf16 (or NULL),
 * out [M,N] (bf16 or fp32), gate_a [N] fp32, gate_b [B,gate_b_stride] fp32, row_req [M] int32,
 * dsig (host, 8 floats) — all device pointers except dsig.  K % 64 == 0, N % 32 == 0. */
int gs_debug_gemm(gs_ctx* ctx, int epi, int M, int N, int K, const void* A, const void* W,
                  const void* bias, void* out, const float* gate_a, const float* gate_b,
                  int gate_b_stride, const int* row_req, const float* dsig_host);
/* The QKV GEMM's bf16 epilogue with the qk-RMSNorm sums of squares: out [M,N] bf16 =
 * A W^T + bias, and for the output columns c < ssq_cols (a multiple of 32), ssq[row * (ssq_cols / 32) + c / 32]
 * = the fp32 sum over that 32-column chunk of (acc + bias)^2.  Device pointers; ssq holds M * ssq_cols / 32
 * floats.  GS_EINVAL for ssq_cols % 32 != 0 or ssq_cols > N. */
int gs_debug_gemm_ssq(gs_ctx* ctx, int M, int N, int K, const void* A, const void* W, const void* bias, void* out,
                      float* ssq, int ssq_cols);
/* Attention over packed requests: Q/K/V/O bf16 [rows, heads, d] with row strides (elements);
 * seq_off/seq_len host int arrays of nreq entries (rows of each request). d in {64, 128}. */
int gs_debug_attention(gs_ctx* ctx, const void* q, const void* k, const void* v, void* o, int heads,
                       int d, int q_rs, int kv_rs, int o_rs, const int* seq_off, const int* seq_len,
                       int nreq);
/* One DiT block (model, layer) at p = 1 on host data: x [N, D] fp32 in/out (rows of the nreq
 * requests concatenated), grids [nreq*3] (F_t, H_t, W_t), tok_lo [nreq] first request-local
 * token of each row segment, n_rows [nreq], t [nreq] timesteps (e = time-embedding(t)).
 * Cross-attention models: prompts = host bf16 [nreq][text_len][text_dim] (one prompt per row
 * segment); NULL otherwise. */
int gs_debug_block(gs_ctx* ctx, int model, int layer, float* x, int nreq, const int* grids,
                   const int* tok_lo, const int* n_rows, const float* t, const void* prompts);
/* Development aid: clock64 stamps written by attention CTAs 0 and 1 (for d = 128 a CTA pair) of
 * head 0 when the environment has GS_ATTN_TRACE=1: [2 CTAs][16 events][32 KV tiles][2 softmax
 * groups]; n <= 2048 entries to host, -1 if larger. */
int gs_debug_attention_trace(unsigned long long* host, size_t n);
/* Development aid (GS_ATTN_TRACE=1): per attention CTA (linear id blockIdx.y * gridDim.x +
 * blockIdx.x < 8192) of the last launch: [entry globaltimer ns, first S issued (leader CTAs),
 * exit, SM id]; n <= 32768 entries to host, -1 if larger. */
int gs_debug_attention_ctatime(unsigned long long* host, size_t n);
/* Time embedding of nreq timesteps: e0 [nreq, D], e [nreq, 6D] fp32 (host outputs). */
int gs_debug_time_embed(gs_ctx* ctx, int model, int nreq, const float* t, float* e0, float* e);

#ifdef __cplusplus
}
#endif
#endif /* GS_H_ */

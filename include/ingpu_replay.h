/*
 * include/ingpu_replay.h -- C-ABI of the B200-native in-GPU experience replay and its
 * device-resident DQN / Double-DQN train step (Parr, "Deep In-GPU Experience Replay",
 * arXiv 1801.03138).
 *
 * Citation keys: P:n = PAPER.md line n (section in brackets); S:n = SPEC.md line n;
 * Qk = reading k of DESIGN.md "Readings of the paper".
 *
 * General conventions
 *   - Every call returns an int status (RPL_OK = 0; > 0 informational; < 0 error).
 *     Argument errors are detected on the host, returned synchronously and leave no
 *     partial effect.  Errors detected on the device (corrupt terminal flag from
 *     a device-sourced add, non-finite loss) set a sticky per-handle flag that the next
 *     rpl_check() reports; rpl_last_error() gives a thread-local message.
 *   - All work is enqueued asynchronously on the handle's CUDA stream (opts.cuda_stream /
 *     cfg.cuda_stream; NULL = legacy default stream) except dqn_get_params,
 *     dqn_debug_export and rpl_check, which synchronise that stream.
 *   - A handle is used by one host thread at a time (external serialisation, S:164,
 *     S:240).
 *   - "device pointer" = memory on the handle's device (e.g. a torch CUDA tensor's
 *     data_ptr()); "host pointer" = ordinary or pinned host memory.
 *   - Nothing here falls back to the CPU: without a usable sm_100 device every call
 *     that needs one returns RPL_ECUDA.
 */
#ifndef INGPU_REPLAY_H
#define INGPU_REPLAY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------------ */
enum {
    RPL_OK = 0,
    RPL_NOT_READY = 1,   /* replay size < burn_in: nothing done, counters unchanged */
    RPL_EINVAL = -1,     /* invalid argument / config / dims / batch                        */
    RPL_ENOMEM = -2,     /* device or pinned allocation failed (message: requested bytes)   */
    RPL_ECORRUPT = -3,   /* terminal flag not in {0,1}                               */
    RPL_ENUMERIC = -4,   /* non-finite loss: that step's update was skipped        */
    RPL_ECUDA = -5,      /* CUDA runtime / launch error                                     */
    RPL_ENCCL = -6,      /* NCCL unavailable or failed                                      */
    RPL_ESTATE = -7      /* call not valid in the handle's state                           */
};

/* where replay_add's inputs live (RPL_DEVICE_DEFER: device, ring write may be deferred) */
enum { RPL_HOST = 0, RPL_DEVICE = 1, RPL_DEVICE_DEFER = 2 };
enum { RPL_ONLINE = 0, RPL_TARGET = 1, RPL_GRAD = 2 };  /* which parameter vector          */
enum { RPL_F32 = 0, RPL_U8 = 1 };                        /* state element type of a replay  */
enum { RPL_SAMPLE_UNIFORM = 0, RPL_SAMPLE_DISTINCT = 1 }; /* sampler of a replay            */
enum { RPL_RING_DEVICE = 0, RPL_RING_HOST = 1, RPL_RING_HOST_BATCH = 2 };  /* where rows live */
enum { RPL_PREC_FP32 = 0, RPL_PREC_TF32 = 1, RPL_PREC_BF16 = 2 };   /* learner precision   */

typedef struct rpl_replay rpl_replay;   /* opaque */
typedef struct rpl_dqn rpl_dqn;         /* opaque */

/* ====================================================================================
 * The replay (P:73 [Methods]: "The Experience Replay API has two methods: adding new
 * experiences, and randomly sampling from the current experiences.")
 * ==================================================================================== */
typedef struct {
    int32_t device;       /* CUDA device ordinal                                            */
    void *cuda_stream;    /* cudaStream_t all work is enqueued on (NULL = default stream)   */
    int64_t burn_in;      /* sampling / training allowed once size >= burn_in (>= 1)  */
    uint64_t seed;        /* Philox key of the sampler (Q3)                                 */
    uint32_t rank;        /* learner rank, < 2^24; selects an independent sampler stream    */
    int64_t max_host_add; /* largest k accepted from host memory per replay_add (pinned
                             staging size); 0 = 65536, capped at 256 MB of staging          */
    int32_t state_dtype;  /* RPL_F32 (default, the paper's float states) or RPL_U8
                             (Atari-shaped byte states; the network input is x = u8/255,
                             SURVEY reading Q27)                                            */
    int32_t sampling;     /* RPL_SAMPLE_UNIFORM (default: uniform with replacement) or
                             RPL_SAMPLE_DISTINCT (P:75's planned switch: the first B distinct
                             values of the same index stream; needs size >= B, B <= 7168)    */
    int32_t state_sharing; /* 1: store one state per experience: the new state of the
                             experience in slot i is the old state of slot i+1; rows hold
                             [s | a | r | terminal] (half the bytes); replay_add ignores
                             s_next (may be NULL); the sampler draws over the size - 1
                             experiences whose successor is stored (all but the newest), at
                             logical position u -> slot (oldest + u) mod capacity            */
    int32_t ring_memory;  /* RPL_RING_DEVICE (default: the method, rows in HBM) or
                             RPL_RING_HOST: the in-RAM comparison mode (
                             P:50): the same rows in pinned, device-mapped host
                             memory, so every sample / gather / train step reads its batch
                             across PCIe -- the per-step transfer the in-GPU replay removes.
                             The kernels, sampler and results are identical.
                             RPL_RING_HOST_BATCH: the paper's in-RAM replay itself ("the
                             RAM variant ... copies sampled batches to the GPU"): rows
                             in ordinary (pageable) host memory written by the CPU on
                             replay_add (RPL_HOST inputs only), every replay_sample /
                             dqn_train_step samples its indices on the CPU (the same Philox
                             stream), gathers the rows on the CPU into pinned staging and
                             copies the batch to the GPU in one H2D transfer of
                             B*(row bytes + 4) bytes (counted in h2d_bytes) before the same
                             train-step kernels run.  fp32 states, uniform or distinct
                             sampling (the CPU draws the same streams: the paper's in-RAM
                             `random.sample` is the distinct rule, reading Q29), one state
                             pair per row, the fast path's net shapes; replay_gather returns
                             RPL_ESTATE                                                      */
    int64_t update_size;  /* 0 (default): every replay_add is one insert, visible at once.
                             U > 0: P:73 block updates ("Experiences are queued in RAM until
                             the queue has enough experiences to update the next block";
                             P:119 uses U = 2,000): RPL_HOST experiences wait in a host queue
                             and every U of them become one insert (one H2D transfer of
                             U*(8*state_dim+9) bytes); queued experiences are not part of
                             the replay (never sampled, not in size / cursor / total) until
                             their block is written or replay_flush_queue writes a partial
                             block.  Device-sourced adds are rejected (EINVAL) in this mode.
                             U <= capacity; U > max_host_add raises max_host_add to U      */
    void *storage;        /* optional caller-owned DEVICE buffer for the ring rows (e.g. a
                             torch tensor): at least replay_ring_bytes() bytes, 256-byte
                             aligned, on opts.device, valid until replay_destroy (which does
                             not free it); zeroed at create.  NULL: the library allocates.
                             Ignored (must be NULL) with RPL_RING_HOST                      */
    size_t storage_bytes; /* its size in bytes                                              */
} rpl_replay_opts;

/* Create an empty FIFO replay of `capacity` experiences whose states are `state_dim`
 * fp32 values ("starts empty"; 1,000,000 x (27+27+3)).  Device layout: one
 * 128-byte-aligned row per slot, [s | s' | a:i32 | r:f32 | terminal:u32 | pad], row
 * stride round_up(2*state_dim+3, 32) floats (256 B for state_dim = 27).  RPL_U8 replays
 * store [s u8 | s' u8 | pad to 16 B | a | r | terminal | pad], row stride
 * round_up(round_up(2*state_dim, 16) + 12, 128) bytes (56,576 B for 84x84x4).
 * opts may be NULL (device 0, default stream, burn_in 1, seed 2, rank 0).
 * Errors: EINVAL (capacity < 1, capacity >= 2^31, state_dim < 1, rank >= 2^24),
 * ENOMEM, ECUDA.  *out owns the device ring until replay_destroy. */
int replay_create(int64_t capacity, int32_t state_dim, const rpl_replay_opts *opts,
                  rpl_replay **out);
/* Bytes of the ring rows replay_create would allocate for these arguments (the size an
 * opts.storage buffer needs).  Errors: EINVAL as replay_create's argument checks. */
int replay_ring_bytes(int64_t capacity, int32_t state_dim, const rpl_replay_opts *opts,
                      size_t *bytes);
int replay_destroy(rpl_replay *replay);

/* Insert k experiences, oldest evicted first: experience j goes to slot
 * (cursor + j) mod capacity; afterwards cursor += k (mod capacity), size = min(size+k,
 * capacity), total += k.  Inputs are SoA: s[k*state_dim], a[k], r[k],
 * s_next[k*state_dim] (fp32, or u8 for RPL_U8 replays), done[k] in {0,1}.
 * mem = RPL_HOST: host pointers, copied into
 * pinned staging before return (the caller may reuse them at once); one H2D transfer of
 * k*(8*state_dim+9) bytes (fp32 states; k*(2*state_dim+9) for u8) is counted in replay_state's
 * h2d_bytes -- the only PCIe traffic of the method.  A deferred host add is read by
 * the device straight from the pinned staging (zero-copy) when the step consumes it; any other
 * host add is copied on the replay's own copy stream, so the transfer overlaps work already
 * queued on the replay's stream, which waits for it before the insert.  Staging is a ring of
 * 2*max_host_add experiences: many small adds can be in flight; an add blocks only when it
 * would overwrite a span the device has not consumed yet.  mem = RPL_DEVICE: device pointers that must stay
 * valid until the stream reaches the insert.  mem = RPL_DEVICE_DEFER: device pointers
 * whose contents must stay valid AND unchanged until the next call on this replay or the
 * next dqn_train_step on it has been reached by the stream.
 * Deferred insert (HOST and DEVICE_DEFER, k <= 4096): the ring write is not a separate
 * kernel; the next fast-path dqn_train_step performs it inside its first kernel, which
 * reads any sampled slot of this insert straight from its source ("read-through"), so
 * the sampled batch is identical.  Any other call on the replay (add, sample, gather,
 * rpl_check) first enqueues the write as an insert kernel.  Observable state (cursor,
 * size, total, and every sample / gather) is the same as with an immediate insert.
 * Errors: EINVAL (k < 0, k > capacity, k > max_host_add for HOST, null pointer with
 * k > 0), ECORRUPT (HOST done[j] > 1; nothing written).  k = 0 is a no-op.
 * A device-sourced done[j] > 1 is written as 1 and raises the sticky ECORRUPT flag. */
int replay_add(rpl_replay *replay, int64_t k, const void *s, const int32_t *a,
               const float *r, const void *s_next, const uint8_t *done, int mem);

/* Caller-owned DEVICE buffers receiving an unpacked batch ("unpacked into old
 * state, new state, action, reward and is_terminal Tensors").  Any pointer may be NULL
 * (that tensor is not written).  s, s_next: [B*state_dim] row-major in the replay's state
 * type (fp32, or u8 for RPL_U8); a: [B] i32; r: [B] fp32; done: [B] u8; idx: [B] i32
 * sampled slot indices. */
typedef struct {
    void *s;
    void *s_next;
    int32_t *a;
    float *r;
    uint8_t *done;
    int32_t *idx;
} rpl_batch;

/* Sample B indices uniformly with replacement from [0, size) (Q1-Q3) and gather
 * + unpack the rows into *out.  Index i of event E is
 *   Philox4x32-10(ctr = (i/2, E_lo, E_hi, (1<<24)|rank), key = (seed_lo, seed_hi)),
 *   u = words (x1:x0) for even i, (x3:x2) for odd i, idx = floor(u * size / 2^64).
 * Consumes one sampler event (E += 1).  RPL_SAMPLE_DISTINCT replays take the first B
 * distinct values of that index stream (position t = index t of the formula above), in
 * stream order.  Returns RPL_NOT_READY (nothing done) while size < burn_in (or, distinct,
 * size < B).  Errors: EINVAL (B < 1; distinct B > 7168). */
int replay_sample(rpl_replay *replay, int32_t batch, const rpl_batch *out);

/* Gather + unpack the rows at the caller's DEVICE indices idx_dev[0..n) (each must be
 * in [0, size); out-of-range indices are clamped and raise the sticky EINVAL flag).
 * No sampler event is consumed.  Used for the gather-bandwidth measurement. */
int replay_gather(rpl_replay *replay, int64_t n, const int32_t *idx_dev, const rpl_batch *out);

/* update_size > 0 only: write the k < U queued experiences as a partial block (a no-op when
 * none wait); *flushed (may be NULL) = k.  replay_queued reports how many wait. */
int replay_flush_queue(rpl_replay *replay, int64_t *flushed);
int replay_queued(const rpl_replay *replay, int64_t *queued);

/* Host mirror of the ring state; no synchronisation. */
int replay_size(const rpl_replay *replay, int64_t *size);
int replay_state(const rpl_replay *replay, int64_t *cursor, int64_t *size, uint64_t *total,
                 uint64_t *events, uint64_t *h2d_bytes);

/* ====================================================================================
 * The DQN learner: the whole train step runs on the device with no input
 * copied from the host.
 * ==================================================================================== */
typedef struct {
    int32_t device;
    void *cuda_stream;
    int32_t state_dim;    /* D (27 for Melee)                                          */
    int32_t n_actions;    /* |A| <= 32 (Q16)                                                 */
    int32_t dueling;      /* 0: plain MLP head; 1: dueling V/A streams             */
    int32_t n_hidden;     /* 1..4 shared hidden ReLU layers                                  */
    int32_t hidden[4];    /* widths (<= 4096)                                                */
    int32_t stream;       /* dueling: units per stream (512 in the paper)             */
    int32_t double_dqn;   /* 0: y = r + g(1-d) max_a Q_t(s',a); 1: Double DQN (Q9)    */
    float gamma;          /* discount in [0, 1]                                              */
    float lr;             /* SGD step alpha                                           */
    float huber_kappa;    /* Huber threshold (> 0); +INFINITY gives 1/2 delta^2 = P:90      */
    int64_t sync_period;  /* target <- online after step t when t % period == 0;
                             0 = only on sync_target()                                       */
    int32_t max_batch;    /* largest batch dqn_train_step accepts (sizes the workspaces)    */
    int64_t avg_period;   /* data-parallel learners (dqn_attach_nccl): 0 = the gradient is
                             averaged over ranks every step ("synchronized every train
                             step"); K > 0 = each rank applies its own SGD and the online and
                             target parameters are averaged over ranks after every K-th step
                             (P:144's "synchronized periodically" / iterative parameter
                             mixing, reading Q31)                                           */
    int32_t precision;    /* tensor-core products of the fast path and of the wide layer 0:
                             RPL_PREC_FP32 (default): FP32-accurate (3xTF32 / bf16x3 splits,
                             the 1e-5 parity of the north star); RPL_PREC_TF32: one product
                             of tf32-rounded operands (wide layer 0: two bf16 terms of the
                             weights); RPL_PREC_BF16: one product of bf16-rounded operands
                             (a BF16 MMA's numerics; parity 2e-2, north star).  The
                             cooperative (generic) kernel computes in FP32 SIMT in every mode */
} rpl_dqn_config;

/* Number of fp32 parameters of the blob layout:
 *   each shared layer l: W_l [N_l x K_l] row-major, then b_l [N_l];
 *   plain head: W [A x N_last], b [A];
 *   dueling: W_st [2S x N_last] (rows 0..S-1 V stream, S..2S-1 A stream), b_st [2S],
 *            W_hd [(1+A) x S] (row 0 V head over V units, rows 1..A A head over A units),
 *            b_hd [1+A].
 * 140,297 for the paper's net (27 -> 128 -> 2 x 512 -> 1 + 8). */
int dqn_param_count(const rpl_dqn_config *cfg, int64_t *n);

/* Create a learner whose online AND target networks start equal to init_params_host
 * (host blob of dqn_param_count floats).  Errors: EINVAL, ENOMEM, ECUDA. */
int dqn_create(const rpl_dqn_config *cfg, const float *init_params_host, rpl_dqn **out);
int dqn_destroy(rpl_dqn *dqn);

/* One train step on `batch` experiences sampled from `replay` (which must live on the
 * same device and stream):  burn-in gate -> Philox sample (event E of the replay)
 * -> gather -> Q_online(s), Q_target(s') [, Q_online(s')] -> TD target, Huber loss ->
 * backward through the online net -> SGD w -= lr * g -> step t += 1 -> target
 * sync when t % sync_period == 0.  One CUDA-graph launch of the fast path's kernels
 * (four up to B = 512, six tcgen05-based ones from B = 640; one cooperative kernel for other
 * shapes; byte-state wide inputs add their layer-0 tensor-core kernels).  Data-parallel
 * learners (world > 1): the gradient mean -- NCCL all-reduce + SGD, or the
 * peer-memory exchange kernel -- is captured in the same graph on the fast path (launched
 * after the step's kernels otherwise).  loss_dev (nullable, fp32, device memory or pinned
 * host memory -- the latter is written by the device over PCIe from a side branch of the
 * step graph, no copy op; for data-parallel learners the ranks' mean loss) receives the
 * batch-mean Huber loss.  Returns RPL_NOT_READY (nothing enqueued, no counter advanced)
 * while size < burn_in.  Errors: EINVAL (batch < 1 or > max_batch, dims differ from the
 * replay's, different device), ECUDA, ENCCL (an NCCL call failed, or a peer of the
 * peer-memory exchange did not arrive: the update is skipped on every rank). */
int dqn_train_step(rpl_dqn *dqn, rpl_replay *replay, int32_t batch, float *loss_dev);

/* target <- online (bit copy), enqueued on the stream. */
int sync_target(rpl_dqn *dqn);

/* Copy a parameter vector (RPL_ONLINE, RPL_TARGET, or RPL_GRAD = the last step's
 * gradient, all-reduced if attached) to / from host memory (n must equal
 * dqn_param_count).  get synchronises the stream. */
int dqn_get_params(rpl_dqn *dqn, int which, float *host_out, int64_t n);
int dqn_set_params(rpl_dqn *dqn, int which, const float *host_in, int64_t n);

/* Executed train steps t (host mirror). */
int dqn_step_count(const rpl_dqn *dqn, int64_t *steps);

/* Debug export of the last train step's device intermediates (synchronises).  `what`:
 *   RPL_DBG_IDX      [B] i32 sampled indices     RPL_DBG_S / RPL_DBG_S_NEXT [B*D] in the
 *                    replay's state type (f32, or u8 for RPL_U8)
 *   RPL_DBG_A        [B] i32                     RPL_DBG_R [B] f32   RPL_DBG_DONE [B] u8
 *   RPL_DBG_Q        [B*A] f32 Q_online(s)       RPL_DBG_QT_NEXT [B*A] f32 Q_target(s')
 *   RPL_DBG_QO_NEXT  [B*A] f32 Q_online(s') (Double DQN only)
 *   RPL_DBG_Y        [B] f32 TD targets          RPL_DBG_ASTAR [B] i32 (Double DQN)
 *   RPL_DBG_H        [B*H] f32 online-net activations on s over the hidden-unit space
 *                    (shared layers in order, then the stream units [V | A])
 *   RPL_DBG_LOSS     [1] f32
 *   RPL_DBG_TRACE    [8 x 2048 x 8] u64 per-CTA marks of the last step's kernels (only with
 *                    env RPL_TRACE=1): slots 0..3 the four fast-path kernels ([0] start and
 *                    [1] end %globaltimer ns, [2..7] SM cycles since start), 4 / 5 the wide
 *                    layer-0 forward / dW0 kernels ([0..7] %globaltimer ns)
 * `bytes` must equal the size of that array for the last step's batch. */
enum { RPL_DBG_IDX = 0, RPL_DBG_S, RPL_DBG_S_NEXT, RPL_DBG_A, RPL_DBG_R, RPL_DBG_DONE,
       RPL_DBG_Q, RPL_DBG_QT_NEXT, RPL_DBG_QO_NEXT, RPL_DBG_Y, RPL_DBG_ASTAR, RPL_DBG_H,
       RPL_DBG_LOSS, RPL_DBG_TRACE };
int dqn_debug_export(rpl_dqn *dqn, int what, void *host_out, int64_t bytes);

/* ====================================================================================
 * Data-parallel learners ("the agent's model would have to be synchronized every
 * train step"): one process per GPU, each with its own replay shard; the gradient is
 * averaged over ranks with NCCL (ncclAllReduce avg over NVLink/NVSwitch) before SGD.
 * ==================================================================================== */
/* Rank 0 creates an NCCL unique id (128 bytes) to broadcast (e.g. torch.distributed). */
int rpl_nccl_unique_id(void *out128);
/* Join the communicator; from then on dqn_train_step all-reduces the gradient. */
int dqn_attach_nccl(rpl_dqn *dqn, int32_t rank, int32_t world, const void *id128);

/* Peer-memory data parallelism within one node (<= 8 ranks, GPUs with peer access over
 * NVLink): the gradient mean and the SGD run in one kernel that reads every rank's gradient
 * from its memory (no NCCL call; P:144 per-step sync).  dqn_peer_handle allocates this
 * learner's exchange buffer (two gradient slots + a flag word) and writes its 64-byte
 * cudaIpcMemHandle to handle_out; after every rank has its peers' handles (e.g. all-gathered
 * with torch.distributed), dqn_attach_peers(rank, world, handles[world * 64 bytes]) maps them.
 * From then on dqn_train_step publishes its gradient, waits for every rank's (device-side
 * flags), averages them in rank order (replicas stay bit-identical) and updates; gradients
 * longer than 2^20 words are averaged reduce-scatter style (each rank averages 1/world of
 * them and stores that slice into every rank's mean buffer) before the update.  Every rank
 * must call dqn_train_step the same number of times.  Errors: EINVAL, ESTATE (no handle yet,
 * NCCL attached, or avg_period > 0), ECUDA (IPC mapping). */
int dqn_peer_handle(rpl_dqn *dqn, void *handle_out);
int dqn_attach_peers(rpl_dqn *dqn, int32_t rank, int32_t world, const void *handles);
/* Undo dqn_attach_peers (synchronises; the exchange buffer stays for a later attach).  A rank
 * whose peer did not arrive within ~10 s skips that step's update and reports RPL_ENCCL at the
 * next synchronising call instead of hanging. */
int dqn_detach_peers(rpl_dqn *dqn);

/* Test entry: the peer-memory gradient mean + SGD for `world` ranks emulated by one
 * cooperative launch on the current device (all buffers device memory on it): xbufs[world]
 * exchange buffers of the layout above (stride = their byte size / 4 floats; slot t % 2 holds
 * rank q's gradient and loss, then the [P + 1] mean of the reduce-scatter variant, then the
 * flag area), online / target [world][P], gmean [world][P + 1] outputs,
 * sync_flag (int32, 1 = copy to target), err (sticky word); t > 0.  Synchronises. */
int rpl_dp_emulate(int32_t world, int64_t P, float *xbufs, float *online, float *target,
                   float *gmean, const int32_t *sync_flag, uint32_t *err, float lr, uint64_t t,
                   int32_t reduce_scatter);

/* Synchronise the handle's stream and report (then clear) its sticky device error:
 * RPL_OK, RPL_ECORRUPT, RPL_ENUMERIC or RPL_ECUDA.  handle = rpl_replay* or rpl_dqn*
 * with kind = 0 (replay) or 1 (dqn). */
int rpl_check(void *handle, int kind);
const char *rpl_last_error(void);
/* Number of kernels this library launched in the calling process (launch accounting). */
uint64_t rpl_kernel_launches(void);

/* Measurement entry (the B200 version of P:119-125 / Fig. 3, cost per add vs update size):
 * n_calls consecutive replay_add(replay, k, s, a, r, s_next, done, mem) calls with the same
 * k-experience inputs, then a synchronisation of the replay's stream; *seconds = the host
 * wall time of the whole loop (no per-call binding overhead).  Stops at the first non-OK
 * status and returns it.  Inputs as replay_add's. */
int rpl_time_adds(rpl_replay *replay, int64_t n_calls, int64_t k, const void *s, const int32_t *a,
                  const float *r, const void *s_next, const uint8_t *done, int mem, double *seconds);

#ifdef __cplusplus
}
#endif
#endif /* INGPU_REPLAY_H */

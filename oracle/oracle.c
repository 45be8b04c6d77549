/*
 * oracle/oracle.c -- the CPU ORACLE for the in-GPU experience-replay DQN train step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` legs may load this library.  The product path
 * (paper_1801_03138_b200/) never imports, links or calls it, and it shares no code,
 * header, table or constant generator with the CUDA path.
 *
 * Plain, slow, single-threaded C.  Floating point is IEEE double (the paper stores
 * fp32 "floats"; the oracle accumulates in fp64 so the fp32 kernels are compared
 * against a more accurate result).  Every function follows the passage it cites.
 *
 * Citation keys:  P:n = /root/reference/PAPER.md line n (section in brackets),
 *                 S:n = /root/reference/SPEC.md line n,
 *                 Qk  = reading k in DESIGN.md section "Readings of the paper".
 *
 * Pins: every function here is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py
 * (Philox known-answer vectors, FIFO brute force, closed forms, finite differences,
 * torch float64 autograd, the paper's worked numbers).  See DESIGN.md "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3").
 * The paper samples "integers uniformly" with TF's random op (P:75 [Methods]); the
 * north star fixes a counter-based Philox generator (reading Q3).
 * ---------------------------------------------------------------------------------- */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

static void philox_round(uint32_t c[4], const uint32_t k[2])
{
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += PHILOX_W0; k[1] += PHILOX_W1; }   /* key bumped between rounds */
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* ------------------------------------------------------------------------------------
 * Uniform with-replacement sampling of B indices in [0, n)  (P:75 [Methods]: "sampling
 * integers uniformly between 0 and the current experience replay size"; readings Q1-Q3).
 * Index i uses Philox call j = i/2 with counter (j, E_lo, E_hi, (TAG_SAMPLE<<24)|rank) and
 * key (seed_lo, seed_hi); words (x0,x1) for even i, (x2,x3) for odd i; u = hi<<32|lo;
 * idx = floor(u * n / 2^64).
 * ---------------------------------------------------------------------------------- */
void oracle_sample_indices(uint64_t seed, uint32_t rank, uint64_t event, int64_t n,
                           int32_t batch, int32_t *idx)
{
    for (int32_t i = 0; i < batch; ++i) {
        uint32_t ctr[4] = {(uint32_t)(i / 2), (uint32_t)event, (uint32_t)(event >> 32),
                           (ORACLE_TAG_SAMPLE << 24) | (rank & 0xFFFFFFu)};
        uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        uint32_t x[4];
        oracle_philox4x32_10(ctr, key, x);
        uint64_t u = (i % 2 == 0) ? (((uint64_t)x[1] << 32) | x[0])
                                  : (((uint64_t)x[3] << 32) | x[2]);
        unsigned __int128 prod = (unsigned __int128)u * (unsigned __int128)(uint64_t)n;
        idx[i] = (int32_t)(uint64_t)(prod >> 64);
    }
}

/* Distinct sampling ("I plan on switching back to sampling distinct integers", i.e.
 * the in-RAM random.sample semantics): the first `batch` DISTINCT values
 * of the same uniform index stream, in stream order (reading Q29).  Needs n >= batch. */
int oracle_sample_distinct(uint64_t seed, uint32_t rank, uint64_t event, int64_t n,
                           int32_t batch, int32_t *idx)
{
    if (n < batch) return ORACLE_EINVAL;
    int32_t count = 0;
    for (int64_t t = 0; count < batch; ++t) {
        int32_t v;
        uint32_t ctr[4] = {(uint32_t)(t / 2), (uint32_t)event, (uint32_t)(event >> 32),
                           (ORACLE_TAG_SAMPLE << 24) | (rank & 0xFFFFFFu)};
        uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        uint32_t x[4];
        oracle_philox4x32_10(ctr, key, x);
        uint64_t u = (t % 2 == 0) ? (((uint64_t)x[1] << 32) | x[0]) : (((uint64_t)x[3] << 32) | x[2]);
        v = (int32_t)(uint64_t)(((unsigned __int128)u * (unsigned __int128)(uint64_t)n) >> 64);
        int seen = 0;
        for (int32_t j = 0; j < count && !seen; ++j) seen = idx[j] == v;
        if (!seen) idx[count++] = v;
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------------------
 * The replay: ONE packed array of C rows x (2D+3) floats, exactly the paper's layout
 * (P:71 [Methods]: "the experience replay Variable has shape 1,000,000 by 57"; action and
 * is_terminal "are cast to floats when added ... and cast back ... when sampling").
 * Field order [s | s' | a | r | terminal].  FIFO with a fixed capacity that starts
 * empty (P:44 [Related Work], P:73 [Methods]).
 * ---------------------------------------------------------------------------------- */
int oracle_ring_init(oracle_ring *ring, int64_t capacity, int32_t state_dim)
{
    if (capacity < 1 || state_dim < 1) return ORACLE_EINVAL;
    ring->capacity = capacity;
    ring->state_dim = state_dim;
    ring->row_width = 2 * state_dim + 3;
    ring->rows = (float *)calloc((size_t)capacity * (size_t)ring->row_width, sizeof(float));
    if (!ring->rows) return ORACLE_ENOMEM;
    ring->cursor = 0;
    ring->size = 0;
    ring->total = 0;
    ring->events = 0;
    ring->distinct = 0;
    ring->shared = 0;
    return ORACLE_OK;
}

/* Shared-state storage ("the new state of an experience is the old state of the next
 * experience.  So, by only storing one state per experience, and modifying the sample
 * operations, ..."; reading Q30): rows [s | a | r | terminal] (D+3
 * floats), the new state of the experience in slot i is the old state of slot (i+1) mod C,
 * and the sampler draws over the size-1 experiences whose successor is stored -- every one
 * but the newest -- at logical position u, slot (oldest + u) mod C.  Only on an empty ring. */
int oracle_ring_set_shared(oracle_ring *ring)
{
    if (ring->size != 0) return ORACLE_EINVAL;
    ring->shared = 1;
    ring->row_width = ring->state_dim + 3;
    return ORACLE_OK;
}

void oracle_ring_free(oracle_ring *ring)
{
    free(ring->rows);
    ring->rows = NULL;
}

/* add k experiences one at a time, oldest evicted first.  k > capacity is
 * rejected before any write (reading Q6). */
int oracle_ring_add(oracle_ring *ring, int64_t k, const float *s, const int32_t *a,
                    const float *r, const float *s_next, const uint8_t *done)
{
    const int32_t D = ring->state_dim;
    if (k < 0 || k > ring->capacity) return ORACLE_EINVAL;
    for (int64_t j = 0; j < k; ++j)
        if (done[j] > 1) return ORACLE_ECORRUPT;
    const int32_t sc = ring->shared ? D : 2 * D;   /* first scalar column */
    for (int64_t j = 0; j < k; ++j) {
        float *row = ring->rows + ring->cursor * ring->row_width;
        for (int32_t d = 0; d < D; ++d) row[d] = s[j * D + d];
        if (!ring->shared)   /* shared: the next experience's s is this one's s' */
            for (int32_t d = 0; d < D; ++d) row[D + d] = s_next[j * D + d];
        row[sc] = (float)a[j];               /* "cast to floats when added" */
        row[sc + 1] = r[j];
        row[sc + 2] = done[j] ? 1.0f : 0.0f;
        ring->cursor = (ring->cursor + 1) % ring->capacity;
        if (ring->size < ring->capacity) ring->size += 1;
        ring->total += 1;
    }
    return ORACLE_OK;
}

/* ---- P:73 block-update queue ------------------------------------------------------------ */
int oracle_queue_init(oracle_queue *q, int64_t update_size, int32_t state_dim)
{
    if (update_size < 1 || state_dim < 1) return ORACLE_EINVAL;
    q->update_size = update_size;
    q->queued = 0;
    q->state_dim = state_dim;
    q->s = (float *)calloc((size_t)update_size * state_dim, sizeof(float));
    q->s_next = (float *)calloc((size_t)update_size * state_dim, sizeof(float));
    q->r = (float *)calloc((size_t)update_size, sizeof(float));
    q->a = (int32_t *)calloc((size_t)update_size, sizeof(int32_t));
    q->done = (uint8_t *)calloc((size_t)update_size, 1);
    if (!q->s || !q->s_next || !q->r || !q->a || !q->done) return ORACLE_ENOMEM;
    return ORACLE_OK;
}

void oracle_queue_free(oracle_queue *q)
{
    free(q->s); free(q->s_next); free(q->r); free(q->a); free(q->done);
    q->s = q->s_next = q->r = NULL;
    q->a = NULL;
    q->done = NULL;
}

/* append the k experiences one at a time; whenever U are waiting they become the next block
 * (one oracle_ring_add of U).  done[j] > 1 anywhere rejects the whole call before any append;
 * k > capacity is rejected as for oracle_ring_add.  s_next may be NULL for a shared ring. */
int oracle_queue_add(oracle_queue *q, oracle_ring *ring, int64_t k, const float *s,
                     const int32_t *a, const float *r, const float *s_next, const uint8_t *done)
{
    const int32_t D = q->state_dim;
    if (k < 0 || k > ring->capacity || D != ring->state_dim) return ORACLE_EINVAL;
    for (int64_t j = 0; j < k; ++j)
        if (done[j] > 1) return ORACLE_ECORRUPT;
    for (int64_t j = 0; j < k; ++j) {
        const int64_t t = q->queued;
        for (int32_t d = 0; d < D; ++d) q->s[t * D + d] = s[j * D + d];
        for (int32_t d = 0; d < D; ++d) q->s_next[t * D + d] = s_next ? s_next[j * D + d] : 0.0f;
        q->a[t] = a[j];
        q->r[t] = r[j];
        q->done[t] = done[j];
        q->queued = t + 1;
        if (q->queued == q->update_size) {
            const int rc = oracle_ring_add(ring, q->update_size, q->s, q->a, q->r, q->s_next, q->done);
            if (rc != ORACLE_OK) return rc;
            q->queued = 0;
        }
    }
    return ORACLE_OK;
}

/* write the k < U waiting experiences as a partial block; returns k (>= 0) or an error */
int64_t oracle_queue_flush(oracle_queue *q, oracle_ring *ring)
{
    const int64_t k = q->queued;
    if (k == 0) return 0;
    const int rc = oracle_ring_add(ring, k, q->s, q->a, q->r, q->s_next, q->done);
    if (rc != ORACLE_OK) return rc;
    q->queued = 0;
    return k;
}

/* gather the rows idx[0..B) and unpack them into five tensors ("the sampled
 * experiences are unpacked into old state, new state, action, reward and is_terminal").
 * Physical slot = logical index (reading Q4). */
int oracle_ring_gather(const oracle_ring *ring, int32_t batch, const int32_t *idx, float *s,
                       int32_t *a, float *r, float *s_next, uint8_t *done)
{
    const int32_t D = ring->state_dim;
    const int32_t sc = ring->shared ? D : 2 * D;
    for (int32_t i = 0; i < batch; ++i) {
        if (idx[i] < 0 || idx[i] >= ring->size) return ORACLE_EINVAL;
        const float *row = ring->rows + (int64_t)idx[i] * ring->row_width;
        for (int32_t d = 0; d < D; ++d) s[i * D + d] = row[d];
        if (ring->shared) {
            /* the experience must have a stored successor: not the newest slot */
            const int64_t newest = (ring->cursor + ring->capacity - 1) % ring->capacity;
            if (idx[i] == newest) return ORACLE_EINVAL;
            const float *nxt = ring->rows + ((int64_t)idx[i] + 1) % ring->capacity * ring->row_width;
            for (int32_t d = 0; d < D; ++d) s_next[i * D + d] = nxt[d];
        } else {
            for (int32_t d = 0; d < D; ++d) s_next[i * D + d] = row[D + d];
        }
        a[i] = (int32_t)row[sc];             /* "cast back to their appropriate types" */
        r[i] = row[sc + 1];
        float t = row[sc + 2];
        if (t != 0.0f && t != 1.0f) return ORACLE_ECORRUPT;
        done[i] = (uint8_t)(t == 1.0f);
    }
    return ORACLE_OK;
}

/* sample = burn-in gate, B uniform indices from event E, gather ("Training is
 * skipped during this burn-in phase").  During burn-in nothing advances (Q5). */
int oracle_ring_sample(oracle_ring *ring, int64_t burn_in, uint64_t seed, uint32_t rank,
                       int32_t batch, int32_t *idx, float *s, int32_t *a, float *r,
                       float *s_next, uint8_t *done)
{
    if (ring->size < burn_in || ring->size < 1) return ORACLE_NOT_READY;
    /* shared states: the newest experience has no stored successor yet (reading Q30) */
    const int64_t n = ring->shared ? ring->size - 1 : ring->size;
    if (n < 1) return ORACLE_NOT_READY;
    if (ring->distinct) {
        if (n < batch) return ORACLE_NOT_READY;   /* reading Q29 */
        oracle_sample_distinct(seed, rank, ring->events, n, batch, idx);
    } else {
        oracle_sample_indices(seed, rank, ring->events, n, batch, idx);
    }
    if (ring->shared) {   /* logical position u -> slot (oldest + u) mod C */
        const int64_t oldest = ring->size < ring->capacity ? 0 : ring->cursor;
        for (int32_t i = 0; i < batch; ++i) idx[i] = (int32_t)((oldest + idx[i]) % ring->capacity);
    }
    ring->events += 1;
    return oracle_ring_gather(ring, batch, idx, s, a, r, s_next, done);
}

/* ------------------------------------------------------------------------------------
 * Byte-state replay (SURVEY config 5: 84x84x4 uint8 Atari-shaped states; the paper's own
 * rows are floats).  Same FIFO, sampler and gather as above over
 * separate arrays; the network input is x = u8 / 255 (reading Q27, oracle_u8_input).
 * ---------------------------------------------------------------------------------- */
int oracle_ring_u8_init(oracle_ring_u8 *ring, int64_t capacity, int32_t state_dim)
{
    if (capacity < 1 || state_dim < 1) return ORACLE_EINVAL;
    ring->capacity = capacity;
    ring->state_dim = state_dim;
    ring->s = (uint8_t *)calloc((size_t)capacity * (size_t)state_dim, 1);
    ring->s_next = (uint8_t *)calloc((size_t)capacity * (size_t)state_dim, 1);
    ring->a = (int32_t *)calloc((size_t)capacity, sizeof(int32_t));
    ring->r = (float *)calloc((size_t)capacity, sizeof(float));
    ring->done = (uint8_t *)calloc((size_t)capacity, 1);
    ring->cursor = 0;
    ring->size = 0;
    ring->total = 0;
    ring->events = 0;
    ring->distinct = 0;
    ring->shared = 0;
    if (!ring->s || !ring->s_next || !ring->a || !ring->r || !ring->done) {
        oracle_ring_u8_free(ring);
        return ORACLE_ENOMEM;
    }
    return ORACLE_OK;
}

void oracle_ring_u8_free(oracle_ring_u8 *ring)
{
    free(ring->s); free(ring->s_next); free(ring->a); free(ring->r); free(ring->done);
    ring->s = ring->s_next = ring->done = NULL;
    ring->a = NULL;
    ring->r = NULL;
}

int oracle_ring_u8_add(oracle_ring_u8 *ring, int64_t k, const uint8_t *s, const int32_t *a,
                       const float *r, const uint8_t *s_next, const uint8_t *done)
{
    const int64_t D = ring->state_dim;
    if (k < 0 || k > ring->capacity) return ORACLE_EINVAL;
    for (int64_t j = 0; j < k; ++j)
        if (done[j] > 1) return ORACLE_ECORRUPT;
    for (int64_t j = 0; j < k; ++j) {
        const int64_t c = ring->cursor;
        memcpy(ring->s + c * D, s + j * D, (size_t)D);
        if (!ring->shared) memcpy(ring->s_next + c * D, s_next + j * D, (size_t)D);
        ring->a[c] = a[j];
        ring->r[c] = r[j];
        ring->done[c] = done[j];
        ring->cursor = (ring->cursor + 1) % ring->capacity;
        if (ring->size < ring->capacity) ring->size += 1;
        ring->total += 1;
    }
    return ORACLE_OK;
}

int oracle_ring_u8_gather(const oracle_ring_u8 *ring, int32_t batch, const int32_t *idx,
                          uint8_t *s, int32_t *a, float *r, uint8_t *s_next, uint8_t *done)
{
    const int64_t D = ring->state_dim;
    for (int32_t i = 0; i < batch; ++i) {
        if (idx[i] < 0 || idx[i] >= ring->size) return ORACLE_EINVAL;
        const int64_t c = idx[i];
        memcpy(s + (int64_t)i * D, ring->s + c * D, (size_t)D);
        if (ring->shared) {   /* the next experience's old state (reading Q30) */
            if (c == (ring->cursor + ring->capacity - 1) % ring->capacity) return ORACLE_EINVAL;
            memcpy(s_next + (int64_t)i * D, ring->s + (c + 1) % ring->capacity * D, (size_t)D);
        } else {
            memcpy(s_next + (int64_t)i * D, ring->s_next + c * D, (size_t)D);
        }
        a[i] = ring->a[c];
        r[i] = ring->r[c];
        done[i] = ring->done[c];
    }
    return ORACLE_OK;
}

int oracle_ring_u8_sample(oracle_ring_u8 *ring, int64_t burn_in, uint64_t seed, uint32_t rank,
                          int32_t batch, int32_t *idx, uint8_t *s, int32_t *a, float *r,
                          uint8_t *s_next, uint8_t *done)
{
    if (ring->size < burn_in || ring->size < 1) return ORACLE_NOT_READY;
    const int64_t n = ring->shared ? ring->size - 1 : ring->size;   /* reading Q30 */
    if (n < 1) return ORACLE_NOT_READY;
    if (ring->distinct) {
        if (n < batch) return ORACLE_NOT_READY;   /* reading Q29 */
        oracle_sample_distinct(seed, rank, ring->events, n, batch, idx);
    } else {
        oracle_sample_indices(seed, rank, ring->events, n, batch, idx);
    }
    if (ring->shared) {
        const int64_t oldest = ring->size < ring->capacity ? 0 : ring->cursor;
        for (int32_t i = 0; i < batch; ++i) idx[i] = (int32_t)((oldest + idx[i]) % ring->capacity);
    }
    ring->events += 1;
    return oracle_ring_u8_gather(ring, batch, idx, s, a, r, s_next, done);
}

/* network input of a byte state: x = u8 / 255 (reading Q27), the fp32 nearest the exact
 * quotient (the double quotient rounded once more cannot hit a float tie: u/255 has the
 * non-terminating binary expansion 0.(u)(u)(u)... for 0 < u < 255) */
void oracle_u8_input(int64_t n, const uint8_t *u, float *x)
{
    for (int64_t i = 0; i < n; ++i) x[i] = (float)((double)u[i] / 255.0);
}

/* ------------------------------------------------------------------------------------
 * The Q-network.  Plain MLP (the team's DQN) or the paper's Dueling DQN (P:88,
 * P:92-94 [Deep Q-Network Model]): shared hidden layers, then a V stream and an A stream
 * of `stream` units each, combined as Q(s,a) = V(s) + A(s,a) - (1/|A|) sum_a' A(s,a').
 * ReLU hidden units, linear heads (reading Q13).
 *
 * Parameter blob (both sides read the same blob format):
 *   for each shared/hidden layer l: W_l [N_l x K_l] row-major, b_l [N_l]
 *   plain  : W_out [A x N_last], b_out [A]
 *   dueling: W_st [2S x N_last] (rows 0..S-1 = V stream, S..2S-1 = A stream), b_st [2S],
 *            W_hd [(1+A) x S] (row 0 = V head over the V units, rows 1..A = A head over
 *            the A units), b_hd [1+A]
 * ---------------------------------------------------------------------------------- */
static int net_valid(const oracle_net *net)
{
    if (net->state_dim < 1 || net->n_actions < 1 || net->n_hidden < 1 || net->n_hidden > 4)
        return 0;
    for (int l = 0; l < net->n_hidden; ++l)
        if (net->hidden[l] < 1) return 0;
    if (net->dueling && net->stream < 1) return 0;
    return 1;
}

int64_t oracle_param_count(const oracle_net *net)
{
    if (!net_valid(net)) return -1;
    int64_t P = 0, K = net->state_dim;
    for (int l = 0; l < net->n_hidden; ++l) {
        P += (int64_t)net->hidden[l] * K + net->hidden[l];
        K = net->hidden[l];
    }
    if (net->dueling) {
        P += 2 * (int64_t)net->stream * K + 2 * net->stream;
        P += (int64_t)(1 + net->n_actions) * net->stream + (1 + net->n_actions);
    } else {
        P += (int64_t)net->n_actions * K + net->n_actions;
    }
    return P;
}

/* number of ReLU units of one forward pass (the "hidden unit space": the shared layers in
 * order, then for dueling the 2S stream units [V | A]) */
int64_t oracle_hidden_units(const oracle_net *net)
{
    int64_t H = 0;
    for (int l = 0; l < net->n_hidden; ++l) H += net->hidden[l];
    if (net->dueling) H += 2 * net->stream;
    return H;
}


/* Activations of one forward pass of one sample. */
typedef struct {
    double *z;     /* pre-activations of all hidden units (hidden-unit space)          */
    double *h;     /* activations: h = z where the unit is on, else 0                   */
    uint8_t *on;   /* ReLU decision per hidden unit: z > 0, or the replayed decision    */
    double *head;  /* plain: Q[A]; dueling: [V, A_1..A_A]                                */
    double *q;     /* Q[A]                                                              */
} fwd_state;

/* one dense layer out[n] = b[n] + sum_k W[n,k] in[k], followed by ReLU (reading Q13) */
static void dense_relu(const double *W, const double *b, const double *in, int64_t N, int64_t K,
                       const uint8_t *mask, double *z, double *h, uint8_t *on)
{
    for (int64_t n = 0; n < N; ++n) {
        double acc = b[n];
        for (int64_t k = 0; k < K; ++k) acc += W[n * K + k] * in[k];
        z[n] = acc;
        on[n] = mask ? (mask[n] != 0) : (acc > 0.0);
        h[n] = on[n] ? acc : 0.0;
    }
}

/* forward one state x[D] through params theta.  If mask != NULL it gives the
 * ReLU decision of every hidden unit (decision replay, reading Q25); else z > 0. */
static void forward_one(const oracle_net *net, const double *theta, const double *x,
                        const uint8_t *mask, fwd_state *st)
{
    const int A = net->n_actions;
    const double *p = theta;
    const double *in = x;
    int64_t K = net->state_dim, off = 0;
    for (int l = 0; l < net->n_hidden; ++l) {
        const int64_t N = net->hidden[l];
        dense_relu(p, p + N * K, in, N, K, mask ? mask + off : NULL, st->z + off, st->h + off,
                   st->on + off);
        p += N * K + N;
        in = st->h + off;
        off += N;
        K = N;
    }
    if (!net->dueling) {
        const double *W = p, *b = p + (int64_t)A * K;
        for (int a = 0; a < A; ++a) {
            double acc = b[a];
            for (int64_t k = 0; k < K; ++k) acc += W[a * K + k] * in[k];
            st->head[a] = acc;
            st->q[a] = acc;
        }
        return;
    }
    /* the two streams of `stream` units each, both fed by the last shared layer */
    const int64_t S = net->stream;
    dense_relu(p, p + 2 * S * K, in, 2 * S, K, mask ? mask + off : NULL, st->z + off,
               st->h + off, st->on + off);
    p += 2 * S * K + 2 * S;
    const double *hv = st->h + off, *ha = st->h + off + S;
    const double *Whd = p, *bhd = p + (1 + A) * S;
    /* V(s) = w_V . h_V + b_V */
    double V = bhd[0];
    for (int64_t u = 0; u < S; ++u) V += Whd[u] * hv[u];
    st->head[0] = V;
    /* A(s,a) = w_a . h_A + b_a */
    double mean = 0.0;
    for (int a = 0; a < A; ++a) {
        double acc = bhd[1 + a];
        for (int64_t u = 0; u < S; ++u) acc += Whd[(1 + a) * S + u] * ha[u];
        st->head[1 + a] = acc;
        mean += acc;
    }
    mean /= (double)A;
    /* Q(s,a) = V(s) + A(s,a) - (1/|A|) sum_a' A(s,a') */
    for (int a = 0; a < A; ++a) st->q[a] = V + st->head[1 + a] - mean;
}

/* backward of one dense+ReLU layer: dz = dh * relu'(z); gW += dz in^T; gb += dz;
 * din += W^T dz (if din != NULL) */
static void dense_relu_backward(const double *W, const double *in, int64_t N, int64_t K,
                                const uint8_t *on, const double *dh, double *gW, double *gb,
                                double *din)
{
    for (int64_t n = 0; n < N; ++n) {
        const double dz = on[n] ? dh[n] : 0.0;
        for (int64_t k = 0; k < K; ++k) gW[n * K + k] += dz * in[k];
        gb[n] += dz;
        if (din)
            for (int64_t k = 0; k < K; ++k) din[k] += dz * W[n * K + k];
    }
}

/* backward of one sample through the online net: accumulate dL/dtheta into grad given
 * dQ[A] = dL/dQ(s, .)  ("nabla_w Q_w(s,a)"; only the online net is trained). */
static void backward_one(const oracle_net *net, const double *theta, const double *x,
                         const fwd_state *st, const double *dQ, double *grad, double *dh)
{
    const int A = net->n_actions;
    const int L = net->n_hidden;
    int64_t poff[4], hoff[4], Kin[4];
    int64_t p = 0, h = 0, K = net->state_dim;
    for (int l = 0; l < L; ++l) {
        poff[l] = p; hoff[l] = h; Kin[l] = K;
        p += (int64_t)net->hidden[l] * K + net->hidden[l];
        h += net->hidden[l];
        K = net->hidden[l];
    }
    const int64_t H = oracle_hidden_units(net);
    for (int64_t i = 0; i < H; ++i) dh[i] = 0.0;
    const double *hlast = st->h + hoff[L - 1];
    double *dhlast = dh + hoff[L - 1];

    if (!net->dueling) {
        const double *W = theta + p;
        double *gW = grad + p, *gb = grad + p + (int64_t)A * K;
        for (int a = 0; a < A; ++a) {
            for (int64_t k = 0; k < K; ++k) gW[a * K + k] += dQ[a] * hlast[k];
            gb[a] += dQ[a];
            for (int64_t k = 0; k < K; ++k) dhlast[k] += dQ[a] * W[a * K + k];
        }
    } else {
        const int64_t S = net->stream;
        const int64_t pst = p, phd = p + 2 * S * K + 2 * S;
        /* combine backward: dV = sum_a dQ_a ; dA_a = dQ_a - (1/|A|) sum_a' dQ_a' */
        double dV = 0.0;
        for (int a = 0; a < A; ++a) dV += dQ[a];
        double dA[ORACLE_MAX_ACTIONS];
        for (int a = 0; a < A; ++a) dA[a] = dQ[a] - dV / (double)A;
        const double *Whd = theta + phd;
        double *gWhd = grad + phd, *gbhd = grad + phd + (1 + A) * S;
        const double *hv = st->h + h, *ha = st->h + h + S;
        double *dstream = dh + h;
        for (int64_t u = 0; u < S; ++u) {
            gWhd[u] += dV * hv[u];
            dstream[u] = dV * Whd[u];
        }
        gbhd[0] += dV;
        for (int64_t u = 0; u < S; ++u) dstream[S + u] = 0.0;
        for (int a = 0; a < A; ++a) {
            for (int64_t u = 0; u < S; ++u) {
                gWhd[(1 + a) * S + u] += dA[a] * ha[u];
                dstream[S + u] += dA[a] * Whd[(1 + a) * S + u];
            }
            gbhd[1 + a] += dA[a];
        }
        dense_relu_backward(theta + pst, hlast, 2 * S, K, st->on + h, dstream, grad + pst,
                            grad + pst + 2 * S * K, dhlast);
    }
    for (int l = L - 1; l >= 0; --l) {
        const int64_t N = net->hidden[l];
        const double *in = (l == 0) ? x : st->h + hoff[l - 1];
        dense_relu_backward(theta + poff[l], in, N, Kin[l], st->on + hoff[l], dh + hoff[l],
                            grad + poff[l], grad + poff[l] + N * Kin[l],
                            l > 0 ? dh + hoff[l - 1] : NULL);
    }
}

/* Huber loss h_kappa(delta) (reading Q11); kappa = +inf gives 1/2 delta^2, the P:90 rule */
double oracle_huber(double delta, double kappa)
{
    const double ad = fabs(delta);
    if (isinf(kappa) || ad <= kappa) return 0.5 * delta * delta;
    return kappa * (ad - 0.5 * kappa);
}

/* d h_kappa / d delta = clamp(delta, -kappa, kappa) */
double oracle_huber_grad(double delta, double kappa)
{
    if (isinf(kappa)) return delta;
    if (delta > kappa) return kappa;
    if (delta < -kappa) return -kappa;
    return delta;
}

/* One DQN / Double-DQN semi-gradient evaluation over a sampled batch:
 *   q_i   = Q_online(s_i, a_i)                      (the enumerate-mask gather)
 *   DQN : y_i = r_i + gamma (1-d_i) max_a' Q_target(s'_i, a')          (reading Q9)
 *   DDQN: a*_i = argmax_a' Q_online(s'_i, a')  (lowest index on ties, Q19)
 *         y_i = r_i + gamma (1-d_i) Q_target(s'_i, a*_i)               (Q9)
 *   delta_i = q_i - y_i ;  L = (1/B) sum_i h_kappa(delta_i)            (Q11)
 *   grad = dL/dtheta_online with y held constant (target fixing).
 * Outputs may be NULL except loss and grad. */
int oracle_dqn_loss_grad(const oracle_net *net, const double *online, const double *target,
                         int32_t batch, const float *s, const int32_t *a, const float *r,
                         const float *s_next, const uint8_t *done, double gamma, double kappa,
                         int double_dqn, const uint8_t *mask_override,
                         const int32_t *argmax_override, double *loss, double *grad,
                         double *q_s, double *q_next_target, double *q_next_online, double *y,
                         int32_t *a_star, double *z_online, uint8_t *on_online)
{
    if (!net_valid(net) || batch < 1 || net->n_actions > ORACLE_MAX_ACTIONS) return ORACLE_EINVAL;
    const int A = net->n_actions;
    const int64_t D = net->state_dim;
    const int64_t H = oracle_hidden_units(net);
    const int64_t P = oracle_param_count(net);
    double *buf = (double *)calloc((size_t)(2 * H + 2 * (1 + A) + 2 * A + H + D) * 3, sizeof(double));
    uint8_t *onbuf = (uint8_t *)calloc((size_t)H * 3, 1);
    if (!buf || !onbuf) { free(buf); free(onbuf); return ORACLE_ENOMEM; }
    fwd_state f0 = {buf, buf + H, onbuf, buf + 2 * H, buf + 2 * H + (1 + A)};
    double *b1 = buf + 2 * H + (1 + A) + A;
    fwd_state f1 = {b1, b1 + H, onbuf + H, b1 + 2 * H, b1 + 2 * H + (1 + A)};
    double *b2 = b1 + 2 * H + (1 + A) + A;
    fwd_state f2 = {b2, b2 + H, onbuf + 2 * H, b2 + 2 * H, b2 + 2 * H + (1 + A)};
    double *dh = b2 + 2 * H + (1 + A) + A;
    double *x = dh + H;
    for (int64_t i = 0; i < P; ++i) grad[i] = 0.0;
    double lsum = 0.0;
    int bad_action = 0;
    for (int32_t i = 0; i < batch; ++i) {
        if (a[i] < 0 || a[i] >= A) { bad_action = 1; break; }
        /* target network on s' (frozen weights) */
        for (int64_t d = 0; d < D; ++d) x[d] = (double)s_next[i * D + d];
        forward_one(net, target, x, NULL, &f1);
        double boot;
        if (!double_dqn) {
            boot = f1.q[0];
            for (int k = 1; k < A; ++k) if (f1.q[k] > boot) boot = f1.q[k];
        } else {
            forward_one(net, online, x, NULL, &f2);
            int best = 0;
            for (int k = 1; k < A; ++k) if (f2.q[k] > f2.q[best]) best = k;
            if (argmax_override) best = argmax_override[i];
            if (a_star) a_star[i] = best;
            if (q_next_online) for (int k = 0; k < A; ++k) q_next_online[i * A + k] = f2.q[k];
            boot = f1.q[best];
        }
        if (q_next_target) for (int k = 0; k < A; ++k) q_next_target[i * A + k] = f1.q[k];
        const double yi = (double)r[i] + gamma * (1.0 - (double)done[i]) * boot;
        if (y) y[i] = yi;
        /* online network on s */
        for (int64_t d = 0; d < D; ++d) x[d] = (double)s[i * D + d];
        forward_one(net, online, x, mask_override ? mask_override + (int64_t)i * H : NULL, &f0);
        if (q_s) for (int k = 0; k < A; ++k) q_s[i * A + k] = f0.q[k];
        if (z_online) for (int64_t u = 0; u < H; ++u) z_online[(int64_t)i * H + u] = f0.z[u];
        if (on_online) for (int64_t u = 0; u < H; ++u) on_online[(int64_t)i * H + u] = f0.on[u];
        const double qi = f0.q[a[i]];
        const double delta = qi - yi;
        lsum += oracle_huber(delta, kappa);
        double dQ[ORACLE_MAX_ACTIONS];
        for (int k = 0; k < A; ++k) dQ[k] = 0.0;
        dQ[a[i]] = oracle_huber_grad(delta, kappa) / (double)batch;
        backward_one(net, online, x, &f0, dQ, grad, dh);
    }
    free(buf);
    free(onbuf);
    if (bad_action) return ORACLE_EINVAL;
    *loss = lsum / (double)batch;
    return ORACLE_OK;
}

/* SGD, the paper's update rule w <- w + alpha (y - Q) grad Q, i.e. w <- w - alpha g */
void oracle_sgd(int64_t n, double *w, const double *g, double lr)
{
    for (int64_t i = 0; i < n; ++i) w[i] = w[i] - lr * g[i];
}

/* O6, data-parallel learners ("the model synchronized every train step"; reading
 * Q22/Q23): every rank r evaluates its own batch mean gradient g_r; the ranks' gradients are
 * summed in rank order 0..N-1, divided by N, and the same SGD step w <- w - alpha * mean is
 * applied on every replica.  grads[r] points at rank r's P-word gradient.  mean_out
 * (nullable) receives the mean. */
void oracle_dp_mean_sgd(int32_t world, int64_t n, double *w, const double *const *grads,
                        double lr, double *mean_out)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int32_t r = 0; r < world; ++r) acc += grads[r][i];
        const double g = acc / (double)world;
        if (mean_out) mean_out[i] = g;
        w[i] = w[i] - lr * g;
    }
}

/* ------------------------------------------------------------------------------------
 * A complete learner: burn-in gate, sample, gather, loss/grad, SGD, step counter and the
 * periodic target sync ("updated to have the same weights as the online network once
 * every 10,000 train steps"; reading Q20: after the update of step t when
 * t mod period == 0).  Parameters are kept in fp32 like the device ("floats") and
 * the arithmetic of each step is done in fp64.
 * ---------------------------------------------------------------------------------- */
int oracle_learner_step(oracle_ring *ring, oracle_learner *ln, int32_t batch, double *loss_out,
                        int32_t *idx_out)
{
    const oracle_net *net = &ln->net;
    const int64_t P = oracle_param_count(net);
    const int64_t D = net->state_dim;
    if (ring->state_dim != D || batch < 1) return ORACLE_EINVAL;
    if (ring->size < ln->burn_in || ring->size < 1) return ORACLE_NOT_READY;
    int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * batch);
    float *s = (float *)malloc(sizeof(float) * batch * D);
    float *s2 = (float *)malloc(sizeof(float) * batch * D);
    int32_t *a = (int32_t *)malloc(sizeof(int32_t) * batch);
    float *r = (float *)malloc(sizeof(float) * batch);
    uint8_t *d = (uint8_t *)malloc((size_t)batch);
    double *on = (double *)malloc(sizeof(double) * P);
    double *tg = (double *)malloc(sizeof(double) * P);
    double *g = (double *)malloc(sizeof(double) * P);
    int rc = ORACLE_ENOMEM;
    if (!idx || !s || !s2 || !a || !r || !d || !on || !tg || !g) goto out;
    rc = oracle_ring_sample(ring, ln->burn_in, ln->seed, ln->rank, batch, idx, s, a, r, s2, d);
    if (rc != ORACLE_OK) goto out;
    for (int64_t i = 0; i < P; ++i) { on[i] = ln->online[i]; tg[i] = ln->target[i]; }
    double L;
    rc = oracle_dqn_loss_grad(net, on, tg, batch, s, a, r, s2, d, ln->gamma, ln->kappa,
                              ln->double_dqn, NULL, NULL, &L, g, NULL, NULL, NULL, NULL, NULL,
                              NULL, NULL);
    if (rc != ORACLE_OK) goto out;
    ln->step += 1;
    if (!isfinite(L)) { rc = ORACLE_ENUMERIC; goto out; }   /* params unmodified */
    oracle_sgd(P, on, g, ln->lr);
    for (int64_t i = 0; i < P; ++i) ln->online[i] = (float)on[i];
    if (ln->sync_period > 0 && ln->step % ln->sync_period == 0)
        for (int64_t i = 0; i < P; ++i) ln->target[i] = ln->online[i];
    if (loss_out) *loss_out = L;
    if (idx_out) for (int32_t i = 0; i < batch; ++i) idx_out[i] = idx[i];
out:
    free(idx); free(s); free(s2); free(a); free(r); free(d); free(on); free(tg); free(g);
    return rc;
}

void oracle_sync_target(oracle_learner *ln)
{
    const int64_t P = oracle_param_count(&ln->net);
    for (int64_t i = 0; i < P; ++i) ln->target[i] = ln->online[i];
}

/*
 * oracle/oracle.h -- declarations of the CPU oracle (TEST INFRASTRUCTURE ONLY; see
 * oracle.c).  This header belongs to the oracle alone: the CUDA path never includes it.
 */
#ifndef INGPU_REPLAY_ORACLE_H
#define INGPU_REPLAY_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_OK = 0, ORACLE_NOT_READY = 1, ORACLE_EINVAL = -1, ORACLE_ENOMEM = -2,
       ORACLE_ECORRUPT = -3, ORACLE_ENUMERIC = -4 };

/* Philox counter word 3 = (TAG << 24) | rank (reading Q3) */
enum { ORACLE_TAG_SAMPLE = 1 };
#define ORACLE_MAX_ACTIONS 64

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void oracle_sample_indices(uint64_t seed, uint32_t rank, uint64_t event, int64_t n,
                           int32_t batch, int32_t *idx);
int oracle_sample_distinct(uint64_t seed, uint32_t rank, uint64_t event, int64_t n,
                           int32_t batch, int32_t *idx);

typedef struct {
    int64_t capacity;
    int32_t state_dim;
    int32_t row_width;   /* 2D+3 floats */
    float *rows;         /* capacity x row_width, packed [s | s' | a | r | terminal] */
    int64_t cursor;      /* next slot to write */
    int64_t size;        /* filled slots, <= capacity */
    uint64_t total;      /* experiences ever added */
    uint64_t events;     /* sampler events consumed */
    int32_t distinct;    /* 1: sample distinct indices (oracle_sample_distinct) */
    int32_t shared;      /* 1: shared-state rows [s | a | r | t] (oracle_ring_set_shared) */
} oracle_ring;

int oracle_ring_init(oracle_ring *ring, int64_t capacity, int32_t state_dim);
int oracle_ring_set_shared(oracle_ring *ring);
void oracle_ring_free(oracle_ring *ring);
int oracle_ring_add(oracle_ring *ring, int64_t k, const float *s, const int32_t *a,
                    const float *r, const float *s_next, const uint8_t *done);
int oracle_ring_gather(const oracle_ring *ring, int32_t batch, const int32_t *idx, float *s,
                       int32_t *a, float *r, float *s_next, uint8_t *done);
int oracle_ring_sample(oracle_ring *ring, int64_t burn_in, uint64_t seed, uint32_t rank,
                       int32_t batch, int32_t *idx, float *s, int32_t *a, float *r,
                       float *s_next, uint8_t *done);

/* P:73 block updates: "Experiences are queued in RAM until the queue has enough experiences
 * to update the next block" -- up to update_size experiences wait in front of a ring and are
 * written to it as one block; queued experiences are not part of the replay */
typedef struct {
    int64_t update_size; /* U: block size */
    int64_t queued;      /* experiences waiting, < U after every call */
    int32_t state_dim;
    float *s, *s_next, *r;
    int32_t *a;
    uint8_t *done;
} oracle_queue;

int oracle_queue_init(oracle_queue *q, int64_t update_size, int32_t state_dim);
void oracle_queue_free(oracle_queue *q);
int oracle_queue_add(oracle_queue *q, oracle_ring *ring, int64_t k, const float *s,
                     const int32_t *a, const float *r, const float *s_next, const uint8_t *done);
int64_t oracle_queue_flush(oracle_queue *q, oracle_ring *ring);

/* byte-state replay (SURVEY config 5) */
typedef struct {
    int64_t capacity;
    int32_t state_dim;
    uint8_t *s, *s_next; /* capacity x state_dim */
    int32_t *a;
    float *r;
    uint8_t *done;
    int64_t cursor, size;
    uint64_t total, events;
    int32_t distinct;    /* 1: sample distinct indices (oracle_sample_distinct) */
    int32_t shared;      /* 1: s' = s of the next slot (set on an empty ring) */
} oracle_ring_u8;

int oracle_ring_u8_init(oracle_ring_u8 *ring, int64_t capacity, int32_t state_dim);
void oracle_ring_u8_free(oracle_ring_u8 *ring);
int oracle_ring_u8_add(oracle_ring_u8 *ring, int64_t k, const uint8_t *s, const int32_t *a,
                       const float *r, const uint8_t *s_next, const uint8_t *done);
int oracle_ring_u8_gather(const oracle_ring_u8 *ring, int32_t batch, const int32_t *idx,
                          uint8_t *s, int32_t *a, float *r, uint8_t *s_next, uint8_t *done);
int oracle_ring_u8_sample(oracle_ring_u8 *ring, int64_t burn_in, uint64_t seed, uint32_t rank,
                          int32_t batch, int32_t *idx, uint8_t *s, int32_t *a, float *r,
                          uint8_t *s_next, uint8_t *done);
void oracle_u8_input(int64_t n, const uint8_t *u, float *x);

typedef struct {
    int32_t state_dim;
    int32_t n_actions;
    int32_t dueling;     /* 0 = plain MLP head, 1 = dueling V/A streams */
    int32_t n_hidden;    /* 1..4 shared hidden layers */
    int32_t hidden[4];
    int32_t stream;      /* units per dueling stream (512 in the paper) */
} oracle_net;

int64_t oracle_param_count(const oracle_net *net);
int64_t oracle_hidden_units(const oracle_net *net);
double oracle_huber(double delta, double kappa);
double oracle_huber_grad(double delta, double kappa);
int oracle_dqn_loss_grad(const oracle_net *net, const double *online, const double *target,
                         int32_t batch, const float *s, const int32_t *a, const float *r,
                         const float *s_next, const uint8_t *done, double gamma, double kappa,
                         int double_dqn, const uint8_t *mask_override,
                         const int32_t *argmax_override, double *loss, double *grad,
                         double *q_s, double *q_next_target, double *q_next_online, double *y,
                         int32_t *a_star, double *z_online, uint8_t *on_online);
void oracle_sgd(int64_t n, double *w, const double *g, double lr);
void oracle_dp_mean_sgd(int32_t world, int64_t n, double *w, const double *const *grads,
                        double lr, double *mean_out);

typedef struct {
    oracle_net net;
    float *online;       /* P params, fp32 like the device (caller-owned) */
    float *target;
    double gamma, kappa, lr;
    int32_t double_dqn;
    int64_t burn_in;
    int64_t sync_period; /* 0 = manual sync only */
    uint64_t seed;
    uint32_t rank;
    int64_t step;        /* executed train steps */
} oracle_learner;

int oracle_learner_step(oracle_ring *ring, oracle_learner *ln, int32_t batch, double *loss_out,
                        int32_t *idx_out);
void oracle_sync_target(oracle_learner *ln);

#ifdef __cplusplus
}
#endif
#endif

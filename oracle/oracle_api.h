/* oracle_api.h -- TEST INFRASTRUCTURE ONLY.
 *
 * One C ABI implemented twice:
 *   ref_*  : oracle/ref_shim.cpp compiled together with the UNMODIFIED reference
 *            sources under /root/reference/proj (recipe: oracle/Makefile, output
 *            oracle/_ref/libpbkd_ref.so).  Only buildable where /root/reference
 *            exists.
 *   orc_*  : oracle/pbkd_oracle.cpp, a from-scratch CPU restatement of the
 *            reference algorithm (every function cites the reference file:line
 *            it restates).  Output oracle/liboracle.so; travels to the GPU box.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference leg
 * may load these libraries.  The product (paper_2012_03096_b200) never does.
 *
 * Conventions: all tensors are fp32 NCHW like pbkd::Tensor4 (tensor.hpp:16-22).
 * Weight vectors are flat concatenations in pbkd::for_each_array /
 * for_each_block_array order (model.cpp:448-483), moving stats included.
 * Functions return 0 on success, non-zero on error (message: X_last_error()).
 */
#ifndef PBKD_ORACLE_API_H
#define PBKD_ORACLE_API_H
#include <stddef.h>
#include <stdint.h>

#ifndef ORC
#define ORC(name) orc_##name
#endif

#ifdef __cplusplus
extern "C" {
#endif
#pragma GCC visibility push(default)

/* Mirrors pbkd::DistillTask (distill.hpp:24-37); kind = CandidateKind ordinal,
 * loss_mode = LossMode ordinal. */
typedef struct {
    int block_index;
    int kind;
    int epochs;
    int eval_every;
    uint64_t seed;
    double threshold;
    int loss_mode;
    float lambda_local;
    float lr;
    float momentum;
    int batch_size;
    long long max_steps;
} orc_task;

typedef struct {
    const float* images; /* count * c*h*w */
    const int* labels;   /* count */
    int count, c, h, w, classes;
} orc_dataset;

typedef struct {
    const int* train_idx;
    int n_train;
    const int* eval_idx;
    int n_eval;
} orc_split;

typedef struct {
    double loss_history[256];
    int n_loss;
    int eval_epoch[256];
    double eval_acc[256];
    int n_eval;
    double final_local_loss;
    double best_eval;
    int failed;
    char failure[256];
} orc_result;

const char* ORC(last_error)(void);

/* tensor.hpp:94-99 */
uint64_t ORC(mix_seed)(uint64_t a, uint64_t b);
/* std::shuffle(idx, mt19937_64(seed)) as in distill.cpp:198-200 */
void ORC(shuffle)(int* idx, int n, uint64_t seed);
/* dataset.cpp:136-164; train/eval buffers must hold n ints */
int ORC(stratified_split)(const int* labels, int n, double eval_fraction, uint64_t seed,
                          int* train_out, int* n_train, int* eval_out, int* n_eval);
/* dataset.cpp:52-84 (3x16x16 stripes) */
int ORC(synthetic_dataset)(int count, uint64_t seed, int threads, float* images, int* labels);

/* scheduler.cpp:43-102.  out_ids holds the concatenated per-worker lists,
 * out_counts[worker_count] their lengths. */
int ORC(round_robin)(const int* ids, int n, int workers, int* out_ids, int* out_counts);
int ORC(wfd)(const int* ids, const double* weights, int n, int workers, int* out_ids,
             int* out_counts, double* predicted_makespan);

/* model spec (model.cpp:225-344) + init_weights (model.cpp:421-425) */
int ORC(teacher_num_floats)(const char* spec, size_t* n);
int ORC(teacher_init)(const char* spec, uint64_t seed, float* out, size_t cap);
int ORC(teacher_num_blocks)(const char* spec, int* n);
/* per-block cost: total MACs of block k (1-based) by count_block_cost (model.cpp:724-777) */
int ORC(block_macs)(const char* spec, int k, long long* macs);
/* build_candidate (replacement.cpp:36-72) flat block arrays */
int ORC(candidate_num_floats)(int kind, int c_in, int c_out, int stride, size_t* n);
int ORC(build_candidate)(int kind, int c_in, int c_out, int stride, uint64_t seed, float* out,
                         size_t cap);

/* --- kernels, ops.hpp --- */
void ORC(dw_fwd)(const float* x, int n, int c, int h, int w, const float* k, int kk, int stride,
                 int pad, float* y);
void ORC(dw_bwd)(const float* x, int n, int c, int h, int w, const float* k, int kk, int stride,
                 int pad, const float* gy, float* gx, float* gk);
void ORC(pw_fwd)(const float* x, int n, int c, int h, int w, const float* k, int co, int stride,
                 float* y);
void ORC(pw_bwd)(const float* x, int n, int c, int h, int w, const float* k, int co, int stride,
                 const float* gy, float* gx, float* gk);
void ORC(conv_fwd)(const float* x, int n, int c, int h, int w, const float* k, int co, int kk,
                   int stride, int pad, float* y);
void ORC(bn_train_fwd)(const float* x, int n, int c, int h, int w, const float* gamma,
                       const float* beta, float* mm, float* mv, float momentum, float* y,
                       float* xhat, float* inv_std);
void ORC(bn_train_bwd)(const float* xhat, const float* inv_std, const float* gamma,
                       const float* gy, int n, int c, int h, int w, float* gx, float* ggamma,
                       float* gbeta);
void ORC(bn_infer_fwd)(const float* x, int n, int c, int h, int w, const float* gamma,
                       const float* beta, const float* mm, const float* mv, float* y);
float ORC(mse)(const float* s, const float* t, size_t count);
void ORC(mse_bwd)(const float* s, const float* t, size_t count, float scale, float* g);
void ORC(sgd)(float* w, const float* g, float* v, size_t n, float lr, float momentum);

/* --- block / network level --- */
/* prefix_infer (model.cpp:695-704) on a batch x (n images of the network input
 * shape); out_shape receives (n,c,h,w). */
int ORC(prefix_infer)(const char* spec, const float* tw, const float* x, int n, int k,
                      int inclusive, float* out, size_t cap, int* out_shape);
/* block_infer of a candidate block given its flat arrays */
int ORC(candidate_infer)(int kind, int c_in, int c_out, int stride, const float* bw,
                         const float* x, int n, int h, int w, float* out, size_t cap);
/* evaluate_with_student_block (distill.cpp:264-283) */
int ORC(eval_with_student)(const char* spec, const float* tw, const orc_dataset* d,
                           const int* eval_idx, int n_eval, int block_index, int kind,
                           const float* student_w, int batch_size, double* acc);
/* train_block (distill.cpp:135-262); block_w receives the best snapshot */
int ORC(train_block)(const char* spec, const float* tw, const orc_dataset* d, const orc_split* s,
                     const orc_task* t, orc_result* r, float* block_w, size_t cap);
/* train_block plus hist64[n_loss]: each loss_history entry recomputed with
 * every batch's MSE summed in fp64 over the same outputs (restatement only). */
int ORC(train_block_f64)(const char* spec, const float* tw, const orc_dataset* d,
                         const orc_split* s, const orc_task* t, orc_result* r, float* block_w,
                         size_t cap, double* hist64);
/* Step-loop replay through the public block API (test_distill.cpp:93-118
 * pattern): n_steps optimizer steps of the train_block loop (epoch shuffles,
 * batches, max_steps ignored), no baseline/eval.  step_loss[n_steps] gets each
 * batch's float local loss; final_w the student arrays after the last step. */
int ORC(train_replay)(const char* spec, const float* tw, const orc_dataset* d,
                      const orc_split* s, const orc_task* t, int n_steps, float* step_loss,
                      float* final_w, size_t cap);

/* train_replay plus, per step, the MSE of the same student/teacher outputs
 * accumulated in fp64 (the reference's float serial sum carries its own
 * rounding error). */
int ORC(train_replay_f64)(const char* spec, const float* tw, const orc_dataset* d,
                          const orc_split* s, const orc_task* t, int n_steps, float* step_loss,
                          double* step_loss64, float* final_w, size_t cap);

/* The bench workload restated on the CPU: n_tasks blocks trained side by side
 * for n_steps optimizer steps each (the train_replay step loop).  The teacher
 * boundaries are computed ONCE per training sample (inference-mode BN is
 * per-sample, model.cpp:553-557, so prefix_infer/block_infer of a batch equals
 * the per-sample results stacked -- bit for bit) on `threads` host threads,
 * then each task runs on its own thread.  step_loss / step_loss64 are
 * [n_tasks][n_steps]; ck_steps (ascending, each in 1..n_steps) selects the
 * steps after which the student arrays are stored: task i's snapshot c lands
 * at ck_w + w_off[i] + c * (w_off[i+1]-w_off[i]) / n_ck.  Restatement only. */
int ORC(train_replay_multi)(const char* spec, const float* tw, const orc_dataset* d,
                            const orc_split* s, const orc_task* tasks, int n_tasks, int n_steps,
                            const int* ck_steps, int n_ck, int threads, float* step_loss,
                            double* step_loss64, float* ck_w, const size_t* w_off);

/* run_parallel (runtime.cpp:124-243): plan = per-worker task-id lists
 * (plan_ids concatenated, plan_counts[w] ids each), policy = SchedulePolicy
 * ordinal.  results[i] / block_w + w_off[i] receive the i-th result of the
 * gather (ascending block index), best snapshot included. */
int ORC(run_parallel)(const char* spec, const float* tw, const orc_dataset* d, const orc_split* s,
                      const orc_task* tasks, int n_tasks, const int* plan_ids,
                      const int* plan_counts, int workers, int policy, orc_result* results,
                      float* block_w, const size_t* w_off);

#pragma GCC visibility pop
#ifdef __cplusplus
}
#endif
#endif

/* pbkd_b200.h -- C ABI of the B200-native blockwise-distillation path.
 *
 * This is the drop-in boundary for the reference's hot path:
 * extern "C", plain pointers and sizes, no C++ or torch types.  The C++ host
 * API in paper_2012_03096_b200/include/pbkd/*.hpp (same signatures as the
 * reference's include/pbkd/*.hpp) is implemented on top of these calls; other
 * languages bind them directly (INTEGRATION.md shows the ctypes binding).
 *
 * Reference interfaces replaced (file:line in /root/reference/proj):
 *   pbkd_run / pbkd_run_parallel  <- pbkd::train_block   (include/pbkd/distill.hpp:72-73)
 *                                    pbkd::run_parallel  (include/pbkd/runtime.hpp:41-43)
 *   pbkd_eval_with_student        <- pbkd::evaluate_with_student_block (distill.hpp:77-79)
 *   pbkd_prefix_infer             <- pbkd::prefix_infer (model.hpp:184-186)
 *   pbkd_candidate_infer          <- pbkd::block_infer on a candidate (model.hpp:154-155)
 *   pbkd_build_candidate          <- pbkd::build_candidate (replacement.hpp:39)
 *   pbkd_round_robin / pbkd_wfd_bin_pack / pbkd_makespan
 *                                 <- scheduler.hpp:29-38
 *   pbkd_stratified_split, pbkd_epoch_order, pbkd_mix_seed
 *                                 <- dataset.hpp:45, distill.cpp:198-200, tensor.hpp:94-99
 *   pbkd_k_* (device pointers)    <- ops.hpp kernels (depthwise :114-178,
 *                                    pointwise :184-239, sgd :545-558)
 *
 * Layout conventions: host tensors are fp32 NCHW exactly like pbkd::Tensor4
 * (tensor.hpp:16-22); block weight vectors are flat in for_each_block_array
 * order (model.cpp:448-478), moving statistics included.  Kernel-level
 * entry points (pbkd_k_*) take DEVICE pointers in the engine's layout:
 * activations NHWC, depthwise weights [9][C] (tap-major), pointwise [Cout][Cin].
 *
 * Errors: every int-returning call returns 0 on success; otherwise
 * pbkd_last_error() (thread-local) holds the message and
 * pbkd_last_error_kind() the class, which the C++ layer maps back to the
 * reference's exception types (SpecError, ShapeError, out_of_range, ...).
 */
#ifndef PBKD_B200_H
#define PBKD_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBKD_ERR_SPEC 1    /* pbkd::SpecError / std::invalid_argument */
#define PBKD_ERR_SHAPE 2   /* pbkd::ShapeError */
#define PBKD_ERR_RANGE 3   /* std::out_of_range */
#define PBKD_ERR_LOGIC 4   /* std::logic_error */
#define PBKD_ERR_CUDA 5    /* CUDA runtime failure */
#define PBKD_ERR_OTHER 6
#define PBKD_ERR_WEIGHTS 7 /* pbkd::WeightsError (unreadable / inconsistent weight file) */

#define PBKD_RUN_STEP_ONLY 1 /* skip epoch-0 baseline and evaluations */
#define PBKD_RUN_NO_GRAPH 2  /* launch eagerly instead of CUDA graphs */
#define PBKD_RUN_PROFILE 4   /* after the last epoch, replay it once eagerly with an
                                event per launch: per-kernel-class device time and
                                algorithmic bytes / flops (measurement runs only) */

typedef struct pbkd_ctx pbkd_ctx;
typedef struct pbkd_results pbkd_results;

/* Mirrors pbkd::DistillTask (distill.hpp:24-37). kind: CandidateKind ordinal
 * (0 two_layer, 1 three_layer, 2 two_layer_skip, 3 three_layer_skip);
 * loss_mode: 0 local_only, 1 combined. */
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
} pbkd_task;

typedef struct {
    int block_index;
    int failed;
    char kind[32];
    char failure[256];
    int n_loss;
    int n_eval;
    long long n_steps;
    size_t n_block_floats;
    int has_best;
    double final_local_loss;
    double best_eval;
    double wall_time_s;
} pbkd_result_info;

typedef struct {
    double timestamp_s;
    int worker_id;
    int task_id;
    int kind; /* 0 dispatch, 1 task_start, 2 task_end, 3 steal, 4 gather */
} pbkd_trace_event;

const char* pbkd_last_error(void);
int pbkd_last_error_kind(void);
const char* pbkd_version(void);

/* ---- context (one GPU) ------------------------------------------------- */
int pbkd_ctx_create(int device, pbkd_ctx** out);
void pbkd_ctx_destroy(pbkd_ctx* ctx);
/* A context over a GPU list: one engine per device, one
 * in-process NCCL clique (ncclCommInitAll).  pbkd_run_parallel then places
 * worker w on devices[w % n] with a host thread per GPU (runtime.cpp:226-233);
 * teacher / dataset loads go to every device.  Devices must be distinct. */
int pbkd_ctx_create_multi(const int* devices, int n, pbkd_ctx** out);
int pbkd_ctx_device_count(const pbkd_ctx* ctx, int* n);
int pbkd_device_count(int* n);

/* ---- teacher: model spec JSON (reference schema, model.cpp:225-344) ---- */
int pbkd_spec_num_floats(const char* spec_json, size_t* n);
int pbkd_spec_num_blocks(const char* spec_json, int* n);
int pbkd_teacher_load(pbkd_ctx* ctx, const char* spec_json, const float* weights, size_t n);
int pbkd_teacher_init(pbkd_ctx* ctx, const char* spec_json, uint64_t seed); /* init_weights */
int pbkd_teacher_weights(pbkd_ctx* ctx, float* out, size_t cap);

/* ---- PBKD weight files (replaces weights_io.hpp save_weights /
 * load_weights / load_into_network / rebuild_network_from_arrays /
 * file_hash, weights_io.cpp:68-319; byte-identical files) ------------- */
/* the loaded teacher, arrays in network traversal order */
int pbkd_teacher_save_file(pbkd_ctx* ctx, const char* path);
/* teacher of spec_json with its weights from a PBKD file (validated by name / shape) */
int pbkd_teacher_load_file(pbkd_ctx* ctx, const char* spec_json, const char* path);
/* network of spec_json (teacher weights `teacher`, n_teacher floats) with block
 * `block_index` (1-based) replaced by a candidate of `kind` (pbkd_task.kind)
 * whose weights are `block` (n_block floats, for_each_block_array order) */
int pbkd_save_student_network(const char* spec_json, const float* teacher, size_t n_teacher, int block_index,
                              int kind, const float* block, size_t n_block, const char* path);
/* rebuild_network_from_arrays over a PBKD file against spec_json: per block 0 =
 * teacher structure, 1 + kind = replacement candidate; the rebuilt network's
 * arrays into out (cap floats, n_out written) */
int pbkd_load_network_file(const char* spec_json, const char* path, int* block_kinds, int max_blocks, float* out,
                           size_t cap, size_t* n_out);
int pbkd_file_hash(const char* path, uint64_t* out);

/* ---- dataset: images fp32 NCHW in [0,1], labels int -------------------- */
int pbkd_dataset_load(pbkd_ctx* ctx, const float* images, const int* labels, int count, int c,
                      int h, int w, int classes);
int pbkd_dataset_load_device(pbkd_ctx* ctx, const float* d_images, const int* labels, int count,
                             int c, int h, int w, int classes);

/* ---- distillation ------------------------------------------------------ */
/* All tasks train on this context's GPU with train_block semantics. */
int pbkd_run(pbkd_ctx* ctx, const pbkd_task* tasks, int n_tasks, const int* train_idx,
             int n_train, const int* eval_idx, int n_eval, int flags, pbkd_results** out);
/* run_parallel semantics (runtime.cpp:124-243): plan validation (SpecError),
 * per-task failure isolation, results gathered in task-id order, trace.
 * plan_ids holds the concatenated per-worker lists, plan_counts their
 * lengths.  policy: 0 round_robin, 1 wfd, 2 work_stealing. */
int pbkd_run_parallel(pbkd_ctx* ctx, const pbkd_task* tasks, int n_tasks, const int* train_idx,
                      int n_train, const int* eval_idx, int n_eval, int worker_count, int policy,
                      const int* plan_ids, const int* plan_counts, int flags, pbkd_results** out);
int pbkd_run_count(const pbkd_results* r);
int pbkd_run_info(const pbkd_results* r, int i, pbkd_result_info* info);
int pbkd_run_loss_history(const pbkd_results* r, int i, double* out, int cap);
int pbkd_run_eval_history(const pbkd_results* r, int i, int* epochs, double* acc, int cap);
/* which: 0 best-eval snapshot (TrainedBlockResult::block), 1 final weights */
int pbkd_run_block(const pbkd_results* r, int i, int which, float* out, size_t cap);
int pbkd_run_step_losses(const pbkd_results* r, int i, float* out, long long cap);
int pbkd_run_trace(const pbkd_results* r, pbkd_trace_event* out, int cap, int* n);
double pbkd_run_wall_time(const pbkd_results* r);
double pbkd_run_epoch_ms(const pbkd_results* r); /* device time of the training epochs */
void pbkd_run_free(pbkd_results* r);
/* PBKD_RUN_PROFILE results: per kernel class (name), launches, device ms,
 * compulsory fp32 bytes and flops of those launches. */
int pbkd_run_profile_count(const pbkd_results* r);
int pbkd_run_profile_entry(const pbkd_results* r, int i, char* name, size_t cap, int* launches, double* ms,
                           double* bytes, double* flops);
/* Same as pbkd_run; device events bracket epochs >= timed_from_epoch (host
 * gaps between epochs included), read back with pbkd_run_timing. */
int pbkd_run_timed(pbkd_ctx* ctx, const pbkd_task* tasks, int n_tasks, const int* train_idx,
                   int n_train, const int* eval_idx, int n_eval, int flags, int timed_from_epoch,
                   pbkd_results** out);
int pbkd_run_timing(const pbkd_results* r, double* timed_ms, int* timed_epochs,
                    long long* launches, double* epoch_ms, int cap, int* n_epochs);
/* Times one launch of a hot kernel in isolation (roofline evidence):
 * which 0 teacher conv implicit GEMM, 1 pointwise GEMM, 2 depthwise fwd,
 * 3 depthwise bwd (fused), 4 loss + BN-backward sums; shapes from the loaded
 * teacher's largest block at `batch` samples.  Outputs ms per launch and the
 * algorithmic bytes / flops of that launch. */
int pbkd_bench_kernel(pbkd_ctx* ctx, int which, int batch, int iters, double* ms, double* bytes,
                      double* flops);

/* ---- multi-GPU: sample-sharded teacher + NCCL exchange ------------------ */
/* Rank 0 creates the 128-byte NCCL id; the launcher broadcasts it; every rank
 * joins.  pbkd_run_sharded then trains the given (local) tasks while this
 * rank runs the teacher forward once on its shard of the training split for
 * every boundary the blocks in g_blocks (owner g_owner) read, and receives
 * the other shards' rows of the boundaries its own blocks read in one
 * grouped ncclSend/ncclRecv round per run.  virtual_shards > 1 on one GPU
 * computes the boundaries shard by shard; share weights the teacher shards. */
int pbkd_nccl_unique_id(char* out128);
int pbkd_ctx_set_comm(pbkd_ctx* ctx, const char* id128, int rank, int world);
int pbkd_run_sharded(pbkd_ctx* ctx, const pbkd_task* tasks, int n_tasks, const int* train_idx,
                     int n_train, const int* eval_idx, int n_eval, int flags, int timed_from_epoch,
                     const int* g_blocks, const int* g_owner, int n_global, int virtual_shards,
                     const double* share, int n_share, pbkd_results** out);
/* Host-side boundary exchange layout (BoundaryPlan, identical on all ranks):
 * blocks / owners: every distilled block and its owner rank; rows: floats per
 * sample of boundaries 0..max(blocks) (n_rows entries).  What rank src sends
 * rank dst once per run, in issue order: boundary xj[i], first train row
 * xrow0[i], xrows[i] rows (cap entries, *n written); *count = floats;
 * shard_begin receives the world+1 shard bounds.  Exposed for the
 * multi-process plan tests. */
int pbkd_exchange_plan(const int* blocks, const int* owners, int nb, const long long* rows, int n_rows,
                       int world, int n_train, const double* share, int src, int dst, size_t* count,
                       int* xj, int* xrow0, int* xrows, int cap, int* n, int* shard_begin);

/* ---- inference ----------------------------------------------------------- */
int pbkd_prefix_infer(pbkd_ctx* ctx, const float* x, int n, int k, int inclusive, float* out,
                      size_t cap, int* out_shape);
int pbkd_candidate_infer(pbkd_ctx* ctx, int kind, int c_in, int c_out, int stride,
                         const float* block_w, const float* x, int n, int h, int w, float* out,
                         size_t cap);
int pbkd_eval_with_student(pbkd_ctx* ctx, int block_index, int kind, const float* student_w,
                           const int* eval_idx, int n_eval, int batch_size, double* acc);

/* ---- host-side, bit-exact indexing and scheduling ------------------------ */
uint64_t pbkd_mix_seed(uint64_t a, uint64_t b);
int pbkd_stratified_split(const int* labels, int n, double eval_fraction, uint64_t seed,
                          int* train_out, int* n_train, int* eval_out, int* n_eval);
int pbkd_epoch_order(const int* train_idx, int n, uint64_t task_seed, int epoch, int* out);
int pbkd_build_candidate(int kind, int c_in, int c_out, int stride, uint64_t seed, float* out,
                         size_t cap, size_t* n);
int pbkd_round_robin(const int* ids, int n, int workers, int* out_ids, int* out_counts);
int pbkd_wfd_bin_pack(const int* ids, const double* weights, int n, int workers, int* out_ids,
                      int* out_counts, double* predicted_makespan);
int pbkd_makespan(const int* plan_ids, const int* plan_counts, int workers, const int* ids,
                  const double* weights, int n, double* out);
int pbkd_mac_proxy_weights(const char* spec_json, const int* blocks, int n, double* out);

/* ---- kernel level (device pointers, NHWC, ctx stream; synchronous) ------ */
int pbkd_k_dw_fwd(pbkd_ctx* ctx, const float* x, const float* w9c, float* y, int n, int h, int w,
                  int c, int stride, int pad);
/* Fused stride-1 depthwise backward of a unit whose input is
 * relu(gamma*((p-mean)*inv)+beta): writes gy_prev = dX * [bn(p) > 0],
 * the depthwise weight gradient gk[9][c] and the batch-norm sums
 * sum_g[c], sum_gx[c] of gy_prev (ops.hpp:149-178, 333-342, 387-393). */
int pbkd_k_dw_bwd(pbkd_ctx* ctx, const float* gy, const float* p, const float* w9c,
                  const float* mean, const float* inv, const float* gamma, const float* beta,
                  float* gy_prev, float* gk, float* sum_g, float* sum_gx, int n, int h, int w,
                  int c);
int pbkd_k_dw_gk(pbkd_ctx* ctx, const float* gy, const float* x, float* gk, int n, int h, int w,
                 int c, int stride, int pad);
/* y[m][o] = sum_j x[m][j] w[o][j]; optional per-channel sum / sum of squares */
int pbkd_k_pw_fwd(pbkd_ctx* ctx, const float* x, const float* w, float* y, int rows, int cin,
                  int cout, float* col_sum, float* col_sq);
/* gx[m][j] = sum_o gy[m][o] w[o][j];  gw[o][j] = sum_m gy[m][o] x[m][j] */
int pbkd_k_pw_bwd(pbkd_ctx* ctx, const float* x, const float* w, const float* gy, float* gx,
                  float* gw, int rows, int cin, int cout);
int pbkd_k_sgd(pbkd_ctx* ctx, float* w, const float* g, float* v, size_t n, float lr,
               float momentum);
/* host-buffer SGD through the device kernel (pbkd::SgdState::step) */
int pbkd_sgd_host(float* w, const float* g, float* v, size_t n, float lr, float momentum);

/* ---- block / network level (layer-by-layer on the GPU, csrc/netexec.cu) ----
 *
 * A block is described by its layer list (pbkd::LayerParams, model.hpp:40-52)
 * plus its arrays flat in for_each_block_array order (model.cpp:448-478).
 * A network is n_blocks feature blocks followed by the classifier block
 * (layer_counts has n_blocks + 1 entries; a classifier of 0 layers = none),
 * arrays flat in for_each_array order.  spec_kind names each block
 * ("conv3x3", "two_layer", ...; replacement.cpp:78-82 decides which blocks
 * are replacements). */
typedef struct {
    int kind; /* pbkd::LayerKind ordinal (model.hpp:25-35) */
    int in_channels, out_channels, kernel, stride, padding;
    int has_weight, has_bias; /* Add: has_weight = 1x1 stride projection */
} pbkd_layer_desc;

typedef struct {
    int n_blocks;
    const int* layer_counts;        /* n_blocks + 1 (classifier last) */
    const pbkd_layer_desc* layers;  /* all layers, block after block */
    const char* const* spec_kinds;  /* n_blocks + 1 */
    int in_c, in_h, in_w;
} pbkd_net_desc;

typedef struct pbkd_block_cache pbkd_block_cache;

/* block_forward (model.cpp:498-551) on a host NCHW batch x -> y.  train: batch
 * statistics, and the updated moving statistics are written back into
 * arrays; cache (optional) receives the device-side cache block_backward
 * needs. */
int pbkd_block_forward(pbkd_ctx* ctx, const pbkd_layer_desc* layers, int n_layers, float* arrays, size_t n_arrays,
                       const float* x, int n, int c, int h, int w, int train, float* y, size_t y_cap, int* y_shape,
                       pbkd_block_cache** cache);
/* block_backward (model.cpp:559-656).  grads (n_arrays, arrays layout):
 * parameter gradients ACCUMULATED when param_grads; gx (optional, x's shape)
 * the input gradient when need_input_grad.  Errors as the reference
 * (std::logic_error on a cache / mode mismatch). */
int pbkd_block_backward(pbkd_ctx* ctx, const pbkd_layer_desc* layers, int n_layers, const float* arrays,
                        size_t n_arrays, const pbkd_block_cache* cache, const float* gy, int n, int c, int h, int w,
                        int need_input_grad, int param_grads, float* grads, float* gx, size_t gx_cap);
void pbkd_block_cache_free(pbkd_block_cache* cache);

/* ops::mse_local_loss / mse_local_loss_bwd (ops.hpp:518-539), host buffers */
int pbkd_mse_local_loss(pbkd_ctx* ctx, const float* s, const float* t, size_t count, float* loss);
int pbkd_mse_local_loss_bwd(pbkd_ctx* ctx, const float* s, const float* t, size_t count, float scale, float* g);

/* reassemble + finetune / train_teacher in one call (distill.cpp:297-441):
 * the teacher of spec_json with weights teacher_w, blocks[i] replaced by a
 * candidate of kinds[i] whose arrays (for_each_block_array order) follow one
 * another in cand_w; then pbkd_fit_network over the context's dataset.
 * net_out (cap floats) receives the trained network, *n_out its length. */
int pbkd_fit_assembled(pbkd_ctx* ctx, const char* spec_json, const float* teacher_w, size_t n_teacher,
                       const int* blocks, const int* kinds, const float* cand_w, int n_replaced,
                       const int* train_idx, int n_train, const int* eval_idx, int n_eval_idx, int epochs,
                       int freeze_non_replaced, float lr, float momentum, int batch_size, uint64_t seed,
                       int teacher_mode, double* initial_eval, double* final_eval, double* loss_hist,
                       int* eval_epochs, double* eval_acc, int* n_eval, float* net_out, size_t cap, size_t* n_out);

/* ops::softmax_cross_entropy_fwd / _bwd (ops.hpp:474-514): logits / probs
 * [n][k] host row-major; loss = mean NLL; probs optional; g accumulated */
int pbkd_softmax_ce(pbkd_ctx* ctx, const float* logits, int n, int k, const int* labels, float* loss,
                    float* probs);
int pbkd_softmax_ce_bwd(pbkd_ctx* ctx, const float* probs, int n, int k, const int* labels, float scale,
                        float* g);

/* evaluate_network (distill.cpp:286-295) over the context's dataset */
int pbkd_evaluate_network(pbkd_ctx* ctx, const pbkd_net_desc* net, const float* arrays, size_t n_arrays,
                          const int* idx, int n_idx, int batch_size, double* acc);
/* finetune (distill.cpp:325-391; teacher_mode 0) or train_teacher
 * (distill.cpp:393-441; teacher_mode 1, freeze ignored) of a network over the
 * context's dataset.  arrays are updated in place.  loss_hist[epochs],
 * eval_epochs / eval_acc [epochs + 1]; n_eval receives the eval count. */
int pbkd_fit_network(pbkd_ctx* ctx, const pbkd_net_desc* net, float* arrays, size_t n_arrays,
                     const int* train_idx, int n_train, const int* eval_idx, int n_eval_idx, int epochs,
                     int freeze_non_replaced, float lr, float momentum, int batch_size, uint64_t seed,
                     int teacher_mode, double* initial_eval, double* final_eval, double* loss_hist,
                     int* eval_epochs, double* eval_acc, int* n_eval);

#ifdef __cplusplus
}
#endif
#endif

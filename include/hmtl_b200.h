/*
 * hmtl_b200.h -- C ABI of the B200-native multi-task-parallel GNN training step.
 *
 * Drop-in boundary for the reference's hot path (/root/reference/proj, namespace
 * hmtl).  The reference is a header-only C++ template API with no FFI; this
 * C ABI is what its C++ types bind to (see include/hmtl_b200.hpp for the
 * C++ drop-in mirror and INTEGRATION.md for the binding).  Each entry point
 * names the reference interface it replaces.
 *
 * Conventions
 *   - Return value: 0 = ok, 1..6 = hmtl::ErrorCode (hmtl/error.hpp:8-15:
 *     contract=1, io=2, comm=3, data=4, config=5, internal=6).  The message of
 *     the last failure on the calling thread is hmtl_last_error().
 *   - Plain pointers and sizes only.  `stream` is a cudaStream_t passed as
 *     void* (NULL = the context's own stream).  Every device call is
 *     stream-ordered; functions that return data to the host synchronise.
 *   - Parameter blocks use the reference's flat BlockLayout offsets
 *     (hmtl/model.hpp:40-90), so host<->device copies are 1:1 with
 *     ModelT::shared_block()/head_block(k).
 *   - Contexts are not thread-safe: one host thread per GPU.
 *   - There is no CPU fallback: without a CUDA device every device entry
 *     point fails with HMTL_ERR_INTERNAL.
 */
#ifndef HMTL_B200_H
#define HMTL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HMTL_ABI_VERSION 1

enum {
  HMTL_OK = 0,
  HMTL_ERR_CONTRACT = 1,
  HMTL_ERR_IO = 2,
  HMTL_ERR_COMM = 3,
  HMTL_ERR_DATA = 4,
  HMTL_ERR_CONFIG = 5,
  HMTL_ERR_INTERNAL = 6
};

/* ModelHyper, hmtl/model.hpp:17-37 (field for field). */
typedef struct hmtl_hyper {
  int n_species, layers, hidden, head_width, head_depth, n_heads;
  double cutoff;
} hmtl_hyper;

/* data::DatasetSpec, hmtl/dataset.hpp:20-32. */
typedef struct hmtl_dataset_spec {
  int dataset_id;
  int n_elements;
  uint8_t elements[32];
  int n_min, n_max;
  double alpha, sigma;
  double mu[20];
  uint64_t count;
  int64_t structure_seed;
} hmtl_dataset_spec;

/* A batch of AtomisticSample (hmtl/graph.hpp:13-21) in host memory, the
 * input of build_batch (hmtl/graph.hpp:46-48).  n_atoms[G]; species[N];
 * positions[3N]; forces[3N]; energy_per_atom[G]; dataset_id[G]. */
typedef struct hmtl_samples {
  int G, N;
  const int* n_atoms;
  const uint8_t* species;
  const double* positions;
  const double* forces;
  const double* energy_per_atom;
  const uint8_t* dataset_id;
} hmtl_samples;

/* Capacity of one context's device buffers (capacity-padded so a whole step
 * can be captured once in a CUDA graph and replayed for any batch that fits). */
typedef struct hmtl_caps {
  int max_graphs, max_nodes;
  long long max_edges;
} hmtl_caps;

/* SPEC trainer knobs. */
typedef struct hmtl_train_cfg {
  float lr, beta1, beta2, eps, weight_decay, w_energy, w_force;
  int use_graph; /* capture the step in a CUDA graph and replay it */
} hmtl_train_cfg;

/* AdamW state of a checkpoint's blocks (the HMTP resume extension). */
typedef struct hmtl_ckpt_opt {
  uint64_t step;
  const float *m_shared, *v_shared;
  const float* const* m_heads; /* [n_heads] */
  const float* const* v_heads;
} hmtl_ckpt_opt;

typedef struct hmtl_ctx hmtl_ctx;

/* ------------------------------------------------------------ host-only */
int hmtl_abi_version(void);
const char* hmtl_last_error(void);
int hmtl_device_count(void);

/* shared_layout / head_layout, hmtl/model.hpp:56-90: total sizes, entries. */
size_t hmtl_shared_size(const hmtl_hyper* hp);
size_t hmtl_head_size(const hmtl_hyper* hp);
int hmtl_layout_entry(const hmtl_hyper* hp, int shared, int i, char* name, size_t name_cap,
                      size_t* rows, size_t* cols, size_t* offset); /* returns #entries */
/* ModelT ctor init (hmtl/model.hpp:158-167, 211-225): which=-1 shared, k head k. */
int hmtl_init_block(const hmtl_hyper* hp, uint64_t seed, int which, float* out);
/* classify_regime / memory_footprint, hmtl/model.hpp:246-263 (mode 0 serial 1 base 2 taskpar) */
int hmtl_classify_regime(size_t p_s, size_t p_h, int n_h);
size_t hmtl_memory_footprint(size_t p_s, size_t p_h, int n_h, int mode);

/* Synthetic multi-source generator (host input source; data::default5_specs and
 * data::generate_dataset, src/dataset.cpp:106-161, 213-239).  Two-call:
 * with out arrays NULL it reports *G and *N; then fill. */
int hmtl_default5_spec(int id, hmtl_dataset_spec* out);
int hmtl_generate(const hmtl_dataset_spec* spec, uint64_t seed, int* G, int* N, int* n_atoms,
                  uint8_t* species, double* positions, double* forces, double* energy,
                  uint8_t* dataset_id);

/* Head -> rank placement for MTL-par on `world` ranks (generalises
 * Mesh{N x M}, hmtl/mesh.hpp:21-31, to uneven groups).  share[r*n_heads+k]
 * receives the fraction of head k's per-step global batch served by rank r.
 * weights[k] = relative per-head work (e.g. GPUs-per-head at world 8).
 * Returns 0 or HMTL_ERR_CONFIG when the heads cannot be balanced. */
int hmtl_head_placement(int world, int n_heads, const double* weights, double* share);

/* Epoch plan, shuffle_epoch (hmtl/datastore.hpp:48-75, src/datastore.cpp:47-97):
 * rank `rank`'s ordered (dataset, index) list for one epoch, steps * b_local
 * items.  mode 0 = base (one permutation of the mixed set over all `world`
 * ranks), 1 = taskpar (dataset ids[i] dealt only over its serving group
 * members[member_off[i] .. member_off[i+1]), ascending ranks; the reference's
 * Mesh is members of id g = g*M .. g*M+M-1).  Host-only, deterministic
 * (reference RNG streams).  Pass null outputs to query *n_items. */
/* HMTP checkpoints (save_checkpoint / load_checkpoint, src/model_io.cpp:62-118):
 * the reference's v1 body (hyper record, shared + every head block as f64) plus
 * an optional trailing "HMTO" section with the AdamW step and m/v of every
 * block, which the reference's reader ignores.  heads = n_heads x P_h floats. */
int hmtl_checkpoint_write(const char* path, const hmtl_hyper* hp, const float* shared, const float* heads,
                          const hmtl_ckpt_opt* opt);
int hmtl_checkpoint_read_hyper(const char* path, hmtl_hyper* hp, int* has_optimizer);

int hmtl_epoch_plan(int mode, const uint8_t* ids, const uint64_t* counts, int n_datasets, const int* members,
                    const int* member_off, int world, uint64_t seed, int b_local, int rank, uint8_t* out_ds,
                    uint64_t* out_idx, size_t cap, int* steps, size_t* n_items);

/* ------------------------------------------------------------ device */
/* ModelT<float>(hp, seed, owned_heads), hmtl/model.hpp:158: creates the device
 * context on `device`, allocates capacity-padded buffers and initialises the
 * parameters exactly as the reference does. */
int hmtl_ctx_create(int device, const hmtl_hyper* hp, uint64_t seed, const int* owned_heads,
                    int n_owned, const hmtl_caps* caps, hmtl_ctx** out);
void hmtl_ctx_destroy(hmtl_ctx* ctx);
void* hmtl_ctx_stream(hmtl_ctx* ctx);
/* Grow the context's batch capacities to at least `need` in place: parameters,
 * AdamW m/v and step counter, streams, the batch pool and an attached NCCL
 * communicator all survive (the reference's ModelT has no capacities; this is
 * what lets a growing batch keep training state).  No-op when `need` fits. */
int hmtl_ctx_reserve(hmtl_ctx* ctx, const hmtl_caps* need);

/* shared_block()/head_block(k) (hmtl/model.hpp:182-187): host <-> device. */
int hmtl_set_block(hmtl_ctx* ctx, int which, const float* host);
int hmtl_get_block(hmtl_ctx* ctx, int which, float* host);
/* GradientBufferT (hmtl/model.hpp:98-115) of the last backward. */
int hmtl_get_grad(hmtl_ctx* ctx, int which, float* host);
/* Checkpoint a context (all heads owned: single rank or MTL-base) with or
 * without its AdamW state; load the blocks this context owns (shared + owned
 * heads, and the optimizer state when present) from any full checkpoint --
 * every MTL-par rank resumes from one file.  Hyperparameters must match. */
int hmtl_checkpoint_save(hmtl_ctx* ctx, const char* path, int with_optimizer);
int hmtl_checkpoint_load(hmtl_ctx* ctx, const char* path);

/* Batch upload: the samples are packed into one pinned staging arena and
 * copied with one cudaMemcpyAsync (build_batch input, hmtl/graph.hpp:46). */
int hmtl_batch_upload(hmtl_ctx* ctx, const hmtl_samples* s, void* stream);
/* Device-resident batch pool: pack samples once into device memory ... */
/* Periodic batch (no reference support): as batch_upload plus
 * the lattice of every structure, cells[G][3][3] (rows a1, a2, a3, Angstrom).
 * The next build_batch / train_step uses the cell-list neighbour list with
 * periodic images; edges carry their source image (x_src + n1 a1 + n2 a2 +
 * n3 a3), rows sorted by (src, image).  batch_upload switches back. */
int hmtl_batch_upload_pbc(hmtl_ctx* ctx, const hmtl_samples* s, const double* cells, void* stream);
/* image (n1, n2, n3) of every edge of the built batch, 3 ints per edge (syncs) */
int hmtl_batch_edge_images(hmtl_ctx* ctx, int* img);
int hmtl_pool_add(hmtl_ctx* ctx, const hmtl_samples* s, int* slot);
/* ... and bind pool slot `slot` as the current batch (device-to-device). */
int hmtl_pool_bind(hmtl_ctx* ctx, int slot, void* stream);

/* Device-resident sample store (DataStore, hmtl/datastore.hpp:77-115): the
 * pool (samples in order; per dataset, local index = order of appearance) is
 * uploaded to HBM once; store_bind gathers a plan's batch (dataset ids[n],
 * local indices[n]) into the context's batch arena on the device -- the same
 * arena bytes hmtl_batch_upload would pack -- so only 4 B per graph (+ offsets)
 * cross PCIe per step.  Errors as build_batch / fetch_samples. */
typedef struct hmtl_store hmtl_store;
int hmtl_store_create(int device, const hmtl_samples* pool, hmtl_store** out);
int hmtl_store_counts(const hmtl_store* st, uint8_t* ids, uint64_t* counts, int cap, int* n);
int hmtl_store_bind(hmtl_ctx* ctx, hmtl_store* st, const uint8_t* ds, const uint64_t* idx, int n, void* stream);
int hmtl_store_destroy(hmtl_store* st);
/* Sharded store: each rank keeps only its DataStore shard (make_partition +
 * balanced_split, src/datastore.cpp:11-45 / :99-145) and fetch_samples'
 * remote reads (request/response over TCP, src/datastore.cpp:192-248) become
 * one grouped NCCL send/recv per step over NVLink/NVSwitch.
 *   shard_range: balanced_split(count, n)[i] = [begin, end).
 *   create_sharded: collective over the context's world communicator
 *     (hmtl_comm_init first).  `shard` = this rank's samples of every dataset it
 *     serves, dataset by dataset, each its range [begin, end) in index order;
 *     ids/counts/members/member_off = the partition (serving ranks of dataset
 *     d: members[member_off[d] .. member_off[d+1]], ascending).  The atom
 *     counts of every shard are broadcast once (4 B per sample).
 *   fetch: collective; plan_ds/plan_idx = this step's plan rows of EVERY rank
 *     ([world][b_local], hmtl_epoch_plan output); owners push what their peers
 *     need (no request message: the plan is known everywhere), then one kernel
 *     assembles the batch arena -- the same bytes store_bind/batch_upload give. */
int hmtl_shard_range(uint64_t count, int n, int i, uint64_t* begin, uint64_t* end);
int hmtl_store_create_sharded(hmtl_ctx* ctx, const hmtl_samples* shard, const uint8_t* ids, const uint64_t* counts,
                              const int* members, const int* member_off, int n_datasets, hmtl_store** out);
int hmtl_store_fetch(hmtl_ctx* ctx, hmtl_store* st, const uint8_t* plan_ds, const uint64_t* plan_idx, int b_local,
                     void* stream);
/* HMTD sample files (hmtl/sample_io.hpp:9-15) straight into a device store:
 * structure checked on the host as read_sample_file_raw, the raw records
 * uploaded as they are, per-record CRC-32 and the parse into the pool on the
 * GPU.  Errors: io (open, magic, version, truncation, trailing bytes, CRC). */
int hmtl_store_from_hmtd(int device, const char* const* paths, int n_files, hmtl_store** out);
/* Energy alignment (align_energies, src/dataset.cpp:263-356; hmtl/dataset.hpp:62-70),
 * SURVEY.md 8(f)4.  store_align: in place on a device store -- per dataset the
 * per-element offsets mu_hat (least squares of energy_per_atom on the element
 * fractions of the present elements; normal equations accumulated on the GPU in
 * FP64 in a fixed order, solved by the reference's GEPP with column dropping,
 * hmtl/linalg.hpp:11-58), then energy -= sum_atoms (mu_d - mu_ref) / n.  ids[i],
 * offsets[i*20 .. i*20+19] (NaN = absent or dropped element) per dataset in
 * ascending id order (cap entries); skipped = dropped elements, n_skipped.
 * align_energies: the reference's file-level call (HMTD in -> aligned HMTD out). */
int hmtl_store_align(hmtl_store* st, uint8_t ref_dataset_id, uint8_t* ids, double* offsets, int cap,
                     uint8_t* skipped, int* n_skipped);
int hmtl_align_energies(int device, const char* const* files, int n_files, uint8_t ref_dataset_id,
                        const char* const* out_files, uint8_t* ids, double* offsets, int cap, uint8_t* skipped,
                        int* n_skipped);
/* store contents back to host (store order) and its size */
int hmtl_store_download(const hmtl_store* st, int* n_atoms, uint8_t* species, double* positions, double* forces,
                        double* energy, uint8_t* dataset_id);
int hmtl_store_shape(const hmtl_store* st, int* G, long long* N);
/* Host-side HMTD writer/header reader (write_sample_file / read_sample_header,
 * src/sample_io.cpp:104-120, 173-189), byte-compatible with the reference. */
int hmtl_hmtd_write(const char* path, uint8_t dataset_id, uint8_t aligned, const hmtl_samples* s);
int hmtl_hmtd_read_header(const char* path, uint8_t* dataset_id, uint8_t* aligned, uint64_t* count);

/* build_batch<float> on the device (hmtl/graph.hpp:46-83): bit-exact FP64
 * cutoff test, dst-major CSR, reverse-edge permutation, per-graph edge offsets. */
int hmtl_build_batch(hmtl_ctx* ctx, void* stream);
/* build_batch's edge set without a model context (hmtl/graph.hpp:46-83; SURVEY.md
 * 8(b) hmtl_nbr_build): the same bit-exact FP64 cutoff search on `device` as the
 * training step.  *E receives the edge count; edge_dst/edge_src[E] (dst-major,
 * ascending src), edge_offset[G+1], row_ptr[N+1] (CSR by dst) and rev[E] (index
 * of the reverse edge) are filled when non-NULL, provided E <= cap (else
 * HMTL_ERR_CONTRACT with *E set, so a caller can size and retry).  Empty graphs
 * are rejected as build_batch does (hmtl/graph.hpp:56). */
int hmtl_nbr_build(int device, const hmtl_samples* s, double cutoff, long long cap, int* E, int* edge_dst,
                   int* edge_src, int* edge_offset, int* row_ptr, int* rev);
/* n_graphs / n_nodes of the batch last bound (upload, pool, store bind/fetch). */
int hmtl_batch_shape(hmtl_ctx* ctx, int* G, int* N);
/* GraphBatchT edge view (syncs): *E, and optionally edge_dst/edge_src[E], edge_offset[G+1]. */
int hmtl_batch_edges(hmtl_ctx* ctx, int* E, int* edge_dst, int* edge_src, int* edge_offset);

/* ModelT::forward, hmtl/model.hpp:338-488 (cache kept on the device). */
int hmtl_forward(hmtl_ctx* ctx, void* stream);
/* PredictionT (hmtl/model.hpp:92-96), syncs: energy_per_atom[G], forces[3N]. */
int hmtl_predictions(hmtl_ctx* ctx, float* energy, float* forces);
/* SPEC loss: loss on device + upstreams dE[G], dF[3N]. */
int hmtl_loss(hmtl_ctx* ctx, float w_energy, float w_force, void* stream);
int hmtl_read_loss(hmtl_ctx* ctx, float* loss); /* syncs */
/* Pipelined trainer loop: loss_post enqueues the D2H read of the current
 * step's result (loss + error bits, one DevHdr) into pinned ring slot
 * `slot % 8` on `stream` without syncing; loss_wait blocks on that slot only and
 * reports the reference's errors as read_loss does.  A loop can launch step
 * i+1 before reading step i's loss. */
int hmtl_loss_post(hmtl_ctx* ctx, int slot, void* stream);
int hmtl_loss_wait(hmtl_ctx* ctx, int slot, float* loss);
/* ModelT::backward, hmtl/model.hpp:490-625.  d_energy/d_forces are HOST
 * upstreams [G], [3N]; pass NULL for both to use the device upstreams of
 * hmtl_loss. */
int hmtl_backward(hmtl_ctx* ctx, const float* d_energy, const float* d_forces, void* stream);
/* SPEC AdamW over every owned block; step counter internal. */
int hmtl_adamw(hmtl_ctx* ctx, const hmtl_train_cfg* cfg, void* stream);
/* train_step: build_batch -> forward -> loss -> backward
 * -> head-group + global gradient allreduce_mean (when a communicator is
 * attached) -> AdamW.  Stream-ordered; read the loss with hmtl_read_loss. */
int hmtl_train_step(hmtl_ctx* ctx, const hmtl_train_cfg* cfg, void* stream);

/* Per-layer parity probe: copies a named device cache tensor to the host
 * (syncs). names: "h" (layer 0..L: input of layer l, L = final), "P", "z1",
 * "z2", "agg", "vz1", "pooled", "ez" (layer = MLP layer), "Qf", "zf" (layer =
 * MLP layer >= 1), "s", "dE", "dF", "grads" (the whole gradient buffer
 * [shared | owned head slots] of the last backward).  Returns #floats written in *n. */
int hmtl_debug_fetch(hmtl_ctx* ctx, const char* name, int layer, float* host, size_t cap, size_t* n);

/* Benchmark instrumentation: when enabled, every kernel scope records CUDA
 * events on its stream.  Eager steps record plain events; graph steps
 * (use_graph) replay a separately captured, single-stream copy of the step
 * graph whose scopes are external event-record nodes, synchronising after
 * each replay (per-scope times without side-stream contention).
 * report (syncs) writes a JSON array [{"name","calls","ms"}] and resets. */
int hmtl_profile_enable(hmtl_ctx* ctx, int on);
int hmtl_profile_report(hmtl_ctx* ctx, char* json, size_t cap);
/* Kernel nodes in the captured step graph (= kernel launches per graph step),
 * -1 before the first graph capture. */
int hmtl_step_kernel_count(hmtl_ctx* ctx, int* n);
/* Step execution mode: 1 = multi-stream step graph (default: energy head,
 * weight gradients and collectives on side streams), 0 = every kernel on the
 * caller's stream (serialised; per-kernel times are then each kernel's own, as
 * a profiler's launch list sees them).  Drops the captured graph; syncs. */
int hmtl_set_stream_mode(hmtl_ctx* ctx, int multi);
/* Engine tuning: per-CTA phase timestamps (SM clocks, [CTA][32]) written by the
 * most recent fused node-chain launch; needs HMTL_CHAIN_STAMPS at ctx_create. */
int hmtl_debug_chain_stamps(hmtl_ctx* ctx, long long* out, int n);

/* Engine self-test (not on the training path): runs the tcgen05 engines on
 * plain row-major matrices on device 0.  mode 0: C[rows x N] = X[rows x K] B[K x N]
 * (Y = B); mode 1: C[K x N] = X[rows x K]^T Y[rows x N].  variant: debug bits. */
int hmtl_selftest_gemm(int mode, int variant, int rows, int K, int N, const float* X, const float* Y, float* C);
/* Tensor-pipe issue-rate probe (engine design; device 0): SM clocks per MMA of
 * n back-to-back M=128 x N MMAs.  variant: 0 tf32 SS, 1 tf32 A-in-TMEM,
 * 2 bf16 SS, 3 bf16 A-in-TMEM. */
int hmtl_selftest_mma_rate(int variant, int N, int n, float* clk_per_mma);
/* Engine design probe: bytes per SM clock moved into shared memory by bulk copies
 * (mode 0 from global, `stride` bytes between CTAs' sources, 0 = shared source;
 * mode 1 between the CTAs of 2-CTA clusters). */
int hmtl_selftest_ingress(int mode, int grid, long long stride, int total, int chunk, int depth, float* bytes_per_clk);
/* Engine design probe: TMEM accumulator layout of one CTA-pair (cta_group::2) MMA,
 * out = [2 CTAs][128 lanes][32 columns]. */
int hmtl_selftest_pair_layout(int M, int N, float* out);
int hmtl_selftest_time(int mode, int rows, int K, int N, int iters, float* ms);

/* ------------------------------------------------------------ comm (NCCL) */
/* collective::allreduce_mean over RankGroup (hmtl/mesh.hpp:276-278, 312-342),
 * re-implemented as NCCL communicators: one world communicator and one per
 * head split by ncclCommSplit(color = head).  share[] as from
 * hmtl_head_placement decides which heads this rank owns. */
int hmtl_comm_unique_id(uint8_t out[128]);
int hmtl_comm_init(hmtl_ctx* ctx, const uint8_t id[128], int world, int rank);
/* Allreduce the last gradients (head groups, then global) on `stream`. */
int hmtl_comm_sync_grads(hmtl_ctx* ctx, void* stream);
/* Communicator census: world size, this rank, and the size of every head's
 * sub-group (head_sizes[k], 0 = head not owned here; n = entries to fill).  With
 * HMTL_COMM_LOG=1, comm_init prints the same to stderr.  Host waits on a step
 * (read_loss, loss_wait) poll ncclCommGetAsyncError and abort every communicator
 * on an asynchronous error or after HMTL_COMM_TIMEOUT_S seconds (default 600),
 * returning HMTL_ERR_COMM (src/mesh.cpp:142-146, 161-171 timeouts / close). */
int hmtl_comm_info(hmtl_ctx* ctx, int* world, int* rank, int* head_sizes, int n);
/* Per-category byte counters (CommStats, hmtl/mesh.hpp:102-131): [encoder_sync, head_sync]. */
int hmtl_comm_bytes(hmtl_ctx* ctx, uint64_t out[2]);

#ifdef __cplusplus
}
#endif
#endif

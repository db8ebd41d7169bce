/*
 * hmtl_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This header and hmtl_oracle.c restate, in plain C and double precision, the
 * algorithm of the multi-task GNN training step of the reference
 * (/root/reference/proj/include/hmtl/{graph,kernels,model}.hpp and the
 * SPEC-only trainer).  It exists to CHECK the
 * CUDA implementation: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2506_21788_b200/) never links or calls it.
 *
 * Parity pinning: tests/golden/*.npz are produced by the compiled reference
 * itself (oracle/_ref/libhmtl_ref.so, built from /root/reference sources by
 * oracle/Makefile); tests/test_oracle_golden.py checks this restatement
 * against them (bit-exact for the edge set, <=1e-13 relative for FP64 math).
 */
#ifndef HMTL_ORACLE_H
#define HMTL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ModelHyper, /root/reference/proj/include/hmtl/model.hpp:17-37 */
typedef struct {
  int n_species, layers, hidden, head_width, head_depth, n_heads;
  double cutoff;
} ho_hyper;

/* GraphBatchT<double> views, hmtl/graph.hpp:27-42 */
typedef struct {
  int G, N, E;
  const int* graph_offset;        /* G+1 */
  const int* edge_offset;         /* G+1 */
  const double* pos;              /* 3N  */
  const uint8_t* species;         /* N   */
  const int* edge_dst;            /* E   */
  const int* edge_src;            /* E   */
  const uint8_t* dataset_id;      /* G   */
  const double* edge_shift;       /* 3E lattice shift S of the source image (PBC), NULL = none */
} ho_batch;

/* Forward cache (subset of ForwardCacheT, hmtl/model.hpp:117-151).  Every
 * pointer may be NULL (not recorded) except when calling ho_backward, which
 * needs h_in, z1, a1, z2, vz1, vp1, agg, h_final, ez, fz. Layout:
 *   h_in, agg, vz1, vp1 : [L][N][H]
 *   z1, a1, z2, m       : [L][E][H]
 *   h_final             : [N][H]
 *   pooled              : [G][H]            (by graph index)
 *   ez                  : [depth][G][W]     (pre-activation per MLP layer; last layer uses col 0)
 *   fz                  : [depth][E][W]     (same for the force MLP, by edge index)
 *   s                   : [E]               (force edge scalar)
 */
typedef struct {
  double *h_in, *z1, *a1, *z2, *m, *agg, *vz1, *vp1, *h_final, *pooled, *ez, *fz, *s;
} ho_cache;

size_t ho_shared_size(const ho_hyper* hp);
size_t ho_head_size(const ho_hyper* hp);
/* number of layout entries and entry i (name into buf) */
int ho_layout_entries(const ho_hyper* hp, int shared, int i, char* name, size_t name_cap,
                      size_t* rows, size_t* cols, size_t* offset);

/* seed_stream, hmtl/rng.hpp:12-14 */
uint64_t ho_seed_stream(uint64_t master, uint64_t stream_id);
/* ModelT ctor / init_block_, hmtl/model.hpp:158-167, 211-225.  which=-1 shared, k>=0 head k */
void ho_init_block(const ho_hyper* hp, uint64_t seed, int which, double* out);

/* Periodic neighbour list (the reference has no PBC, so this
 * FP64 brute force over lattice images is the builder's own oracle).  cells:
 * [G][3][3], rows = lattice vectors a1, a2, a3.  Edge (i, j, n): source image
 * x_j + S, S = (n1 a1 + n2 a2) + n3 a3 per component, test
 * ((xi - xj) - S)^2 summed as (dx*dx + dy*dy) + dz*dz <= rc^2, self pair
 * (i, i, 0) excluded.  Rows sorted by (src, image key (n1+8)*256+(n2+8)*16+(n3+8)),
 * |n_k| <= 7.  Returns E (count when edge_dst == NULL), -1 empty graph, -2
 * image range exceeded.  img: 3 ints per edge; shift: 3 doubles per edge. */
long ho_build_edges_pbc(int G, const int* n_atoms, const double* pos, const double* cells, double cutoff,
                        int* graph_offset, int* edge_offset, int* edge_dst, int* edge_src, int* img, double* shift);

/* build_batch edge search, hmtl/graph.hpp:46-83. Returns E (count) when
 * edge_dst == NULL, else fills and returns E. -1 on empty graph. */
long ho_build_edges(int G, const int* n_atoms, const double* pos, double cutoff,
                    int* graph_offset, int* edge_offset, int* edge_dst, int* edge_src);

/* ModelT::forward, hmtl/model.hpp:338-488. heads[k] == NULL => head k not owned.
 * Returns 0 ok, 1 contract error (empty batch / unowned head), 6 non-finite. */
int ho_forward(const ho_hyper* hp, const double* shared, const double* const* heads,
               const ho_batch* b, ho_cache* c, double* energy, double* forces);

/* ModelT::backward, hmtl/model.hpp:490-625.  g_shared / g_heads[k] are
 * overwritten (zero_grads + accumulate). */
int ho_backward(const ho_hyper* hp, const double* shared, const double* const* heads,
                const ho_batch* b, const ho_cache* c, const double* d_energy,
                const double* d_forces, double* g_shared, double* const* g_heads);

/* SPEC loss, /root/reference/SPEC.md:383-391 (no reference code). */
double ho_loss(const ho_batch* b, const double* energy, const double* forces,
               const double* label_energy, const double* label_force, double w_e,
               double w_f, double* d_energy, double* d_forces);

/* SPEC AdamW: decoupled decay, bias correction
 * (torch.optim.AdamW ordering; the choice is recorded in DESIGN.md). */
void ho_adamw(double* p, const double* g, double* m, double* v, size_t n, long step,
              double lr, double beta1, double beta2, double eps, double wd);

#ifdef __cplusplus
}
#endif
#endif

/*
 * hmtl_oracle.c -- plain-C, FP64 restatement of the reference training-step
 * math.  TEST INFRASTRUCTURE ONLY (see hmtl_oracle.h): the checker, never the
 * thing measured or shipped.
 *
 * Every loop below keeps the reference's summation order so that the result
 * is bit-identical to ModelT<double> compiled without FMA contraction
 * (reference build flags: -O3 -g, no -march, /root/reference/proj/CMakeLists.txt:10).
 * This file is compiled with -ffp-contract=off for the same reason.
 */
#include "hmtl_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG --- */
/* splitmix64 / seed_stream: hmtl/rng.hpp:10-14 */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t ho_seed_stream(uint64_t master, uint64_t stream_id) {
  return splitmix64(splitmix64(master) ^ splitmix64(stream_id + 1));
}

/* std::mt19937_64 (the engine behind hmtl::Rng, hmtl/rng.hpp:20-77), as
 * specified by the C++ standard [rand.predef]. */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;
static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}
static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ull) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}
/* Rng::uniform (53 bits), hmtl/rng.hpp:26-31 */
static double mt64_uniform(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }

/* --------------------------------------------------------------- layout --- */
/* shared_layout / head_layout, hmtl/model.hpp:56-90 */
typedef struct {
  char name[48];
  size_t rows, cols, offset;
} entry_t;

static int build_layout(const ho_hyper* hp, int shared, entry_t* out, int cap) {
  int n = 0;
  size_t total = 0;
#define ADD(nm, r, c)                                                   \
  do {                                                                  \
    if (n < cap) {                                                      \
      snprintf(out[n].name, sizeof out[n].name, "%s", nm);              \
      out[n].rows = (r);                                                \
      out[n].cols = (c);                                                \
      out[n].offset = total;                                            \
    }                                                                   \
    total += (size_t)(r) * (size_t)(c);                                 \
    ++n;                                                                \
  } while (0)
  const size_t H = (size_t)hp->hidden;
  char nm[48];
  if (shared) {
    ADD("embed", (size_t)hp->n_species, H);
    for (int l = 0; l < hp->layers; ++l) {
      snprintf(nm, sizeof nm, "layer%d.edge.W1", l); ADD(nm, 2 * H + 1, H);
      snprintf(nm, sizeof nm, "layer%d.edge.b1", l); ADD(nm, 1, H);
      snprintf(nm, sizeof nm, "layer%d.edge.W2", l); ADD(nm, H, H);
      snprintf(nm, sizeof nm, "layer%d.edge.b2", l); ADD(nm, 1, H);
      snprintf(nm, sizeof nm, "layer%d.node.W1", l); ADD(nm, 2 * H, H);
      snprintf(nm, sizeof nm, "layer%d.node.b1", l); ADD(nm, 1, H);
      snprintf(nm, sizeof nm, "layer%d.node.W2", l); ADD(nm, H, H);
      snprintf(nm, sizeof nm, "layer%d.node.b2", l); ADD(nm, 1, H);
    }
  } else {
    const char* pre[2] = {"energy", "force"};
    for (int p = 0; p < 2; ++p) {
      size_t in = p == 0 ? H : H + 1;
      for (int i = 0; i < hp->head_depth; ++i) {
        size_t o = (i == hp->head_depth - 1) ? 1 : (size_t)hp->head_width;
        snprintf(nm, sizeof nm, "%s.W%d", pre[p], i); ADD(nm, in, o);
        snprintf(nm, sizeof nm, "%s.b%d", pre[p], i); ADD(nm, 1, o);
        in = o;
      }
    }
  }
#undef ADD
  return n;
}

static size_t layout_total(const ho_hyper* hp, int shared) {
  entry_t e[512];
  int n = build_layout(hp, shared, e, 512);
  return e[n - 1].offset + e[n - 1].rows * e[n - 1].cols;
}
size_t ho_shared_size(const ho_hyper* hp) { return layout_total(hp, 1); }
size_t ho_head_size(const ho_hyper* hp) { return layout_total(hp, 0); }

int ho_layout_entries(const ho_hyper* hp, int shared, int i, char* name, size_t name_cap,
                      size_t* rows, size_t* cols, size_t* offset) {
  entry_t e[512];
  int n = build_layout(hp, shared, e, 512);
  if (i < 0 || i >= n) return n;
  if (name) snprintf(name, name_cap, "%s", e[i].name);
  if (rows) *rows = e[i].rows;
  if (cols) *cols = e[i].cols;
  if (offset) *offset = e[i].offset;
  return n;
}

/* init_block_, hmtl/model.hpp:211-225: biases zero, weights U(-s,s),
 * s = 0.5 for the embedding, 1/sqrt(rows) otherwise; streams
 * seed_stream(seed,0) (shared) and seed_stream(seed,1+k) (head k), :162,:165. */
void ho_init_block(const ho_hyper* hp, uint64_t seed, int which, double* out) {
  entry_t e[512];
  const int shared = which < 0;
  int n = build_layout(hp, shared, e, 512);
  mt64 rng;
  mt64_seed(&rng, ho_seed_stream(seed, shared ? 0 : (uint64_t)(1 + which)));
  memset(out, 0, (e[n - 1].offset + e[n - 1].rows * e[n - 1].cols) * sizeof(double));
  for (int k = 0; k < n; ++k) {
    if (strstr(e[k].name, ".b")) continue;
    double s = (shared && strcmp(e[k].name, "embed") == 0) ? 0.5 : 1.0 / sqrt((double)e[k].rows);
    double* p = out + e[k].offset;
    for (size_t i = 0; i < e[k].rows * e[k].cols; ++i) p[i] = -s + (s - (-s)) * mt64_uniform(&rng);
  }
}

/* ---------------------------------------------------------- graph batch --- */
/* build_batch pair loop, hmtl/graph.hpp:46-83: dst-major (i outer, j inner),
 * FP64 test (dx*dx+dy*dy)+dz*dz <= rc*rc (inclusive, :71), no self edges. */
long ho_build_edges(int G, const int* n_atoms, const double* pos, double cutoff,
                    int* graph_offset, int* edge_offset, int* edge_dst, int* edge_src) {
  const double rc2 = cutoff * cutoff;
  long E = 0;
  int base = 0;
  if (graph_offset) graph_offset[0] = 0;
  if (edge_offset) edge_offset[0] = 0;
  for (int g = 0; g < G; ++g) {
    const int n = n_atoms[g];
    if (n < 1) return -1; /* "build_batch: empty graph rejected", :56 */
    const double* P = pos + 3 * (size_t)base;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        if (i == j) continue;
        double dx = P[3 * i] - P[3 * j];
        double dy = P[3 * i + 1] - P[3 * j + 1];
        double dz = P[3 * i + 2] - P[3 * j + 2];
        if (dx * dx + dy * dy + dz * dz <= rc2) {
          if (edge_dst) {
            edge_dst[E] = base + i;
            edge_src[E] = base + j;
          }
          ++E;
        }
      }
    base += n;
    if (graph_offset) graph_offset[g + 1] = base;
    if (edge_offset) edge_offset[g + 1] = (int)E;
  }
  return E;
}

static void* xmalloc(size_t n) {
  void* p = calloc(n ? n : 1, 1);
  if (!p) abort();
  return p;
}

/* --------------------------------------------------------------- PBC ----- */
static void lat_shift(const double* A, int n1, int n2, int n3, double* S) {
  for (int k = 0; k < 3; ++k) S[k] = ((double)n1 * A[k] + (double)n2 * A[3 + k]) + (double)n3 * A[6 + k];
}
typedef struct { int j, key, n1, n2, n3; } pbc_hit;
static int pbc_cmp(const void* a, const void* b) {
  const pbc_hit *x = (const pbc_hit*)a, *y = (const pbc_hit*)b;
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  return x->key < y->key ? -1 : (x->key > y->key);
}
long ho_build_edges_pbc(int G, const int* n_atoms, const double* pos, const double* cells, double cutoff,
                        int* graph_offset, int* edge_offset, int* edge_dst, int* edge_src, int* img, double* shift) {
  const double rc2 = cutoff * cutoff;
  long E = 0;
  int base = 0;
  if (graph_offset) graph_offset[0] = 0;
  if (edge_offset) edge_offset[0] = 0;
  for (int g = 0; g < G; ++g) {
    const int n = n_atoms[g];
    if (n < 1) return -1;
    const double* A = cells + 9 * (size_t)g;
    const double* P = pos + 3 * (size_t)base;
    /* generous image range: |fractional displacement| + rc / width, from the
       reciprocal rows (f = x A^-1) */
    const double a[3][3] = {{A[0], A[1], A[2]}, {A[3], A[4], A[5]}, {A[6], A[7], A[8]}};
    double c[3][3];
    for (int k = 0; k < 3; ++k) {
      const int u = (k + 1) % 3, v = (k + 2) % 3;
      c[k][0] = a[u][1] * a[v][2] - a[u][2] * a[v][1];
      c[k][1] = a[u][2] * a[v][0] - a[u][0] * a[v][2];
      c[k][2] = a[u][0] * a[v][1] - a[u][1] * a[v][0];
    }
    const double V = a[0][0] * c[0][0] + a[0][1] * c[0][1] + a[0][2] * c[0][2];
    /* per pair, the images whose fractional displacement can be within rc:
       n_k in [floor(fd_k - rc/w_k) - 1, ceil(fd_k + rc/w_k) + 1], fd = f_i - f_j */
    double span[3];
    double* F = xmalloc(sizeof(double) * 3 * (size_t)n);
    for (int k = 0; k < 3; ++k) {
      const double cn = sqrt(c[k][0] * c[k][0] + c[k][1] * c[k][1] + c[k][2] * c[k][2]);
      span[k] = cutoff * cn / fabs(V);
      for (int i = 0; i < n; ++i)
        F[3 * i + k] = (P[3 * i] * c[k][0] + P[3 * i + 1] * c[k][1] + P[3 * i + 2] * c[k][2]) / V;
    }
    size_t cap = 64;
    pbc_hit* hits = xmalloc(sizeof(pbc_hit) * cap);
    for (int i = 0; i < n; ++i) {
      int h = 0;
      for (int j = 0; j < n; ++j) {
        int lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
          const double fd = F[3 * i + k] - F[3 * j + k];
          lo[k] = (int)floor(fd - span[k]) - 1;
          hi[k] = (int)ceil(fd + span[k]) + 1;
        }
        for (int n1 = lo[0]; n1 <= hi[0]; ++n1)
          for (int n2 = lo[1]; n2 <= hi[1]; ++n2)
            for (int n3 = lo[2]; n3 <= hi[2]; ++n3) {
              if (i == j && n1 == 0 && n2 == 0 && n3 == 0) continue;
              double S[3];
              lat_shift(A, n1, n2, n3, S);
              const double dx = (P[3 * i] - P[3 * j]) - S[0];
              const double dy = (P[3 * i + 1] - P[3 * j + 1]) - S[1];
              const double dz = (P[3 * i + 2] - P[3 * j + 2]) - S[2];
              if ((dx * dx + dy * dy) + dz * dz <= rc2) {
                if (abs(n1) > 7 || abs(n2) > 7 || abs(n3) > 7) {
                  free(hits), free(F);
                  return -2;
                }
                if ((size_t)h == cap) {
                  pbc_hit* nh = xmalloc(sizeof(pbc_hit) * cap * 2);
                  memcpy(nh, hits, sizeof(pbc_hit) * cap);
                  free(hits);
                  hits = nh, cap *= 2;
                }
                pbc_hit t = {j, (n1 + 8) * 256 + (n2 + 8) * 16 + (n3 + 8), n1, n2, n3};
                hits[h++] = t;
              }
            }
      }
      qsort(hits, (size_t)h, sizeof(pbc_hit), pbc_cmp);
      for (int q = 0; q < h; ++q) {
        if (edge_dst) {
          edge_dst[E] = base + i;
          edge_src[E] = base + hits[q].j;
          if (img) img[3 * E] = hits[q].n1, img[3 * E + 1] = hits[q].n2, img[3 * E + 2] = hits[q].n3;
          if (shift) lat_shift(A, hits[q].n1, hits[q].n2, hits[q].n3, shift + 3 * E);
        }
        ++E;
      }
    }
    free(hits), free(F);
    base += n;
    if (graph_offset) graph_offset[g + 1] = base;
    if (edge_offset) edge_offset[g + 1] = (int)E;
  }
  return E;
}

/* ------------------------------------------------------------ numcore ----- */
/* Threading (OpenMP, the checker's only concession to full-size parity runs):
 * every parallel loop below splits work so that each output element is still
 * produced by ONE thread with the reference's operation sequence -- rows of y /
 * dx are independent, and accumulations (dW, db, segment sums, scatters) are
 * split by output element with the reduction loop (ascending batch row / edge)
 * kept inside.  Results are therefore bit-identical to the serial loops for any
 * thread count (pinned by tests/test_oracle_golden.py against the reference). */
#define HO_PAR _Pragma("omp parallel for schedule(static)")
#define HO_PAR_DYN _Pragma("omp parallel for schedule(dynamic, 1)")

/* hmtl/kernels.hpp:19-32 */
static void linear_forward(const double* x, size_t batch, size_t in, const double* W,
                           size_t out, const double* bias, double* y) {
  HO_PAR
  for (size_t b = 0; b < batch; ++b) {
    double* yb = y + b * out;
    for (size_t o = 0; o < out; ++o) yb[o] = bias ? bias[o] : 0.0;
    const double* xb = x + b * in;
    for (size_t i = 0; i < in; ++i) {
      const double xi = xb[i];
      const double* Wi = W + i * out;
      for (size_t o = 0; o < out; ++o) yb[o] += xi * Wi[o];
    }
  }
}
/* hmtl/kernels.hpp:37-59 (accumulates into dW/db) */
/* (element (i,o) of dW receives xb[i]*ub[o] for b ascending exactly as the
 * reference's row loop; rows are visited in blocks of 64 so a block of `up`
 * stays cache-resident across a thread's dW rows) */
static void linear_backward(const double* x, size_t batch, size_t in, const double* W,
                            size_t out, const double* up, double* dW, double* db, double* dx) {
  const size_t BB = 64;
  HO_PAR_DYN
  for (size_t i0 = 0; i0 < in; i0 += 8) {
    const size_t i1 = i0 + 8 < in ? i0 + 8 : in;
    for (size_t b0 = 0; b0 < batch; b0 += BB) {
      const size_t b1 = b0 + BB < batch ? b0 + BB : batch;
      for (size_t i = i0; i < i1; ++i) {
        double* dWi = dW + i * out;
        for (size_t b = b0; b < b1; ++b) {
          const double xi = x[b * in + i];
          const double* ub = up + b * out;
          for (size_t o = 0; o < out; ++o) dWi[o] += xi * ub[o];
        }
      }
    }
  }
  for (size_t b = 0; b < batch; ++b) {
    const double* ub = up + b * out;
    for (size_t o = 0; o < out; ++o) db[o] += ub[o];
  }
  if (dx) {
    HO_PAR
    for (size_t b = 0; b < batch; ++b) {
      const double* ub = up + b * out;
      double* dxb = dx + b * in;
      for (size_t i = 0; i < in; ++i) {
        const double* Wi = W + i * out;
        double acc = 0.0;
        for (size_t o = 0; o < out; ++o) acc += ub[o] * Wi[o];
        dxb[i] = acc;
      }
    }
  }
}
/* hmtl/kernels.hpp:62-82 */
static double sigmoid(double x) {
  if (x >= 0.0) {
    double e = exp(-x);
    return 1.0 / (1.0 + e);
  }
  double e = exp(x);
  return e / (1.0 + e);
}
static double silu(double x) { return x * sigmoid(x); }
static double silu_grad(double x) {
  double s = sigmoid(x);
  return s * (1.0 + x * (1.0 - s));
}

/* ------------------------------------------------------------- layouts ---- */
typedef struct {
  size_t off[512];
  size_t rows[512], cols[512];
  int n;
} lay_t;
static void lay_make(const ho_hyper* hp, int shared, lay_t* L) {
  entry_t e[512];
  L->n = build_layout(hp, shared, e, 512);
  for (int i = 0; i < L->n; ++i) {
    L->off[i] = e[i].offset;
    L->rows[i] = e[i].rows;
    L->cols[i] = e[i].cols;
  }
}



/* head MLP forward, mlp_forward_ hmtl/model.hpp:282-306.  `first` is the
 * entry index of <prefix>.W0 in the head layout; entries alternate W,b. */
static void mlp_forward(const ho_hyper* hp, const double* block, const lay_t* L, int first,
                        const double* x, size_t rows, size_t in_dim, double** z_out /*[depth]*/,
                        double** a_out /*[depth]*/, double* out) {
  const int D = hp->head_depth;
  double* cur = xmalloc(rows * in_dim * sizeof(double));
  memcpy(cur, x, rows * in_dim * sizeof(double));
  size_t in = in_dim;
  for (int i = 0; i < D; ++i) {
    int we = first + 2 * i, be = first + 2 * i + 1;
    size_t od = L->cols[we];
    a_out[i] = cur;
    double* z = xmalloc(rows * od * sizeof(double));
    linear_forward(cur, rows, in, block + L->off[we], od, block + L->off[be], z);
    z_out[i] = xmalloc(rows * od * sizeof(double));
    memcpy(z_out[i], z, rows * od * sizeof(double));
    if (i + 1 < D) {
      HO_PAR
      for (size_t t = 0; t < rows * od; ++t) z[t] = silu(z[t]);
    }
    cur = z;
    in = od;
  }
  memcpy(out, cur, rows * sizeof(double)); /* last layer has 1 output */
  free(cur);
}

/* mlp_backward_, hmtl/model.hpp:308-336; returns d(input) [rows x in_dim] */
static double* mlp_backward(const ho_hyper* hp, const double* block, double* gblock,
                            const lay_t* L, int first, size_t rows, double* const* z,
                            double* const* a, const double* d_out) {
  const int D = hp->head_depth;
  double* up = xmalloc(rows * sizeof(double));
  memcpy(up, d_out, rows * sizeof(double));
  for (int i = D - 1; i >= 0; --i) {
    int we = first + 2 * i, be = first + 2 * i + 1;
    size_t od = L->cols[we], in = L->rows[we];
    if (i + 1 < D) {
      HO_PAR
      for (size_t t = 0; t < rows * od; ++t) up[t] = up[t] * silu_grad(z[i][t]);
    }
    double* dx = xmalloc(rows * in * sizeof(double));
    linear_backward(a[i], rows, in, block + L->off[we], od, up, gblock + L->off[we],
                    gblock + L->off[be], dx);
    free(up);
    up = dx;
  }
  return up;
}

/* ------------------------------------------------------------- forward ---- */
int ho_forward(const ho_hyper* hp, const double* shared, const double* const* heads,
               const ho_batch* b, ho_cache* c, double* energy, double* forces) {
  if (b->G <= 0 || b->N <= 0) return 1; /* :341-342 */
  for (int g = 0; g < b->G; ++g)
    if (b->graph_offset[g + 1] - b->graph_offset[g] <= 0) return 1; /* :343-344 */
  for (int g = 0; g < b->G; ++g)
    if (b->dataset_id[g] >= hp->n_heads || !heads[b->dataset_id[g]]) return 1; /* :345-347 */

  const size_t H = (size_t)hp->hidden, N = (size_t)b->N, E = (size_t)b->E, G = (size_t)b->G;
  const size_t W = (size_t)hp->head_width;
  lay_t SL, HL;
  lay_make(hp, 1, &SL);
  lay_make(hp, 0, &HL);

  /* geometry, :354-366 */
  double* d2 = xmalloc(E * sizeof(double));
  double* d = xmalloc(E * sizeof(double));
  double* dvec = xmalloc(3 * E * sizeof(double));
  for (size_t e = 0; e < E; ++e) {
    const double* pi = b->pos + 3 * (size_t)b->edge_dst[e];
    const double* pj = b->pos + 3 * (size_t)b->edge_src[e];
    double dx = pi[0] - pj[0], dy = pi[1] - pj[1], dz = pi[2] - pj[2];
    if (b->edge_shift) { /* periodic image of the source (8(f)4) */
      dx -= b->edge_shift[3 * e], dy -= b->edge_shift[3 * e + 1], dz -= b->edge_shift[3 * e + 2];
    }
    dvec[3 * e] = dx;
    dvec[3 * e + 1] = dy;
    dvec[3 * e + 2] = dz;
    d2[e] = dx * dx + dy * dy + dz * dz;
    d[e] = sqrt(d2[e]);
  }
  /* embedding, :368-372 */
  const double* embed = shared + SL.off[0];
  double* h = xmalloc(N * H * sizeof(double));
  for (size_t i = 0; i < N; ++i)
    for (size_t k = 0; k < H; ++k) h[i * H + k] = embed[(size_t)b->species[i] * H + k];

  const size_t K1 = 2 * H + 1;
  double* u = xmalloc(E * K1 * sizeof(double));
  double* z1 = xmalloc(E * H * sizeof(double));
  double* a1 = xmalloc(E * H * sizeof(double));
  double* z2 = xmalloc(E * H * sizeof(double));
  double* m = xmalloc(E * H * sizeof(double));
  double* agg = xmalloc(N * H * sizeof(double));
  double* v = xmalloc(N * 2 * H * sizeof(double));
  double* vz1 = xmalloc(N * H * sizeof(double));
  double* vp1 = xmalloc(N * H * sizeof(double));
  double* q = xmalloc(N * H * sizeof(double));
  for (int l = 0; l < hp->layers; ++l) {
    const size_t base = 1 + 8 * (size_t)l; /* :378 */
    const double *eW1 = shared + SL.off[base + 0], *eb1 = shared + SL.off[base + 1];
    const double *eW2 = shared + SL.off[base + 2], *eb2 = shared + SL.off[base + 3];
    const double *nW1 = shared + SL.off[base + 4], *nb1 = shared + SL.off[base + 5];
    const double *nW2 = shared + SL.off[base + 6], *nb2 = shared + SL.off[base + 7];
    if (c && c->h_in) memcpy(c->h_in + (size_t)l * N * H, h, N * H * sizeof(double));
    /* message m_ij = phi_e(h_i, h_j, d_ij^2), :388-406 */
    HO_PAR
    for (size_t e = 0; e < E; ++e) {
      double* ue = u + e * K1;
      const double* hd = h + (size_t)b->edge_dst[e] * H;
      const double* hs = h + (size_t)b->edge_src[e] * H;
      for (size_t k = 0; k < H; ++k) ue[k] = hd[k];
      for (size_t k = 0; k < H; ++k) ue[H + k] = hs[k];
      ue[2 * H] = d2[e];
    }
    linear_forward(u, E, K1, eW1, H, eb1, z1);
    HO_PAR
    for (size_t t = 0; t < E * H; ++t) a1[t] = silu(z1[t]);
    linear_forward(a1, E, H, eW2, H, eb2, z2);
    HO_PAR
    for (size_t t = 0; t < E * H; ++t) m[t] = silu(z2[t]);
    /* segment_sum over dst, ascending e: hmtl/kernels.hpp:97-108 (columns split
     * over threads, every column's sum in edge order) */
    memset(agg, 0, N * H * sizeof(double));
    HO_PAR
    for (size_t k0 = 0; k0 < H; k0 += 4) {
      const size_t k1 = k0 + 4 < H ? k0 + 4 : H;
      for (size_t e = 0; e < E; ++e) {
        double* os = agg + (size_t)b->edge_dst[e] * H;
        const double* vr = m + e * H;
        for (size_t k = k0; k < k1; ++k) os[k] += vr[k];
      }
    }
    /* node update with residual, :408-426 */
    for (size_t i = 0; i < N; ++i) {
      for (size_t k = 0; k < H; ++k) v[i * 2 * H + k] = h[i * H + k];
      for (size_t k = 0; k < H; ++k) v[i * 2 * H + H + k] = agg[i * H + k];
    }
    linear_forward(v, N, 2 * H, nW1, H, nb1, vz1);
    for (size_t t = 0; t < N * H; ++t) vp1[t] = silu(vz1[t]);
    linear_forward(vp1, N, H, nW2, H, nb2, q);
    HO_PAR
    for (size_t t = 0; t < N * H; ++t) h[t] += q[t];
    if (c) {
      const size_t oe = (size_t)l * E * H, on = (size_t)l * N * H;
      if (c->z1) memcpy(c->z1 + oe, z1, E * H * sizeof(double));
      if (c->a1) memcpy(c->a1 + oe, a1, E * H * sizeof(double));
      if (c->z2) memcpy(c->z2 + oe, z2, E * H * sizeof(double));
      if (c->m) memcpy(c->m + oe, m, E * H * sizeof(double));
      if (c->agg) memcpy(c->agg + on, agg, N * H * sizeof(double));
      if (c->vz1) memcpy(c->vz1 + on, vz1, N * H * sizeof(double));
      if (c->vp1) memcpy(c->vp1 + on, vp1, N * H * sizeof(double));
    }
  }
  if (c && c->h_final) memcpy(c->h_final, h, N * H * sizeof(double));

  for (size_t g = 0; g < G; ++g) energy[g] = 0.0;
  for (size_t t = 0; t < 3 * N; ++t) forces[t] = 0.0;

  const int D = hp->head_depth;
  const int fe_first = 0, ff_first = 2 * D; /* entry index of energy.W0 / force.W0 */
  int* graphs = xmalloc(G * sizeof(int));
  /* heads in ascending k (std::map), graphs ascending, :430-433 */
  for (int k = 0; k < hp->n_heads; ++k) {
    size_t Gk = 0;
    for (size_t g = 0; g < G; ++g)
      if (b->dataset_id[g] == k) graphs[Gk++] = (int)g;
    if (!Gk) continue;
    const double* block = heads[k];
    /* energy branch: mean pool (sum then * S(1)/S(n)), :443-457 */
    double* pooled = xmalloc(Gk * H * sizeof(double));
    for (size_t gi = 0; gi < Gk; ++gi) {
      int g = graphs[gi];
      int lo = b->graph_offset[g], hi = b->graph_offset[g + 1];
      for (int i = lo; i < hi; ++i)
        for (size_t kk = 0; kk < H; ++kk) pooled[gi * H + kk] += h[(size_t)i * H + kk];
      const double inv = 1.0 / (double)(hi - lo);
      for (size_t kk = 0; kk < H; ++kk) pooled[gi * H + kk] *= inv;
      if (c && c->pooled) memcpy(c->pooled + (size_t)g * H, pooled + gi * H, H * sizeof(double));
    }
    double *ez[64], *ea[64];
    double* eout = xmalloc(Gk * sizeof(double));
    mlp_forward(hp, block, &HL, fe_first, pooled, Gk, H, ez, ea, eout);
    for (size_t gi = 0; gi < Gk; ++gi) energy[graphs[gi]] = eout[gi];
    if (c && c->ez)
      for (int i = 0; i < D; ++i) {
        size_t od = HL.cols[fe_first + 2 * i];
        for (size_t gi = 0; gi < Gk; ++gi)
          for (size_t o = 0; o < od; ++o)
            c->ez[((size_t)i * G + graphs[gi]) * W + o] = ez[i][gi * od + o];
      }
    for (int i = 0; i < D; ++i) free(ez[i]), free(ea[i]);
    free(eout);
    free(pooled);

    /* force branch: s_e = psi([h_i + h_j, d]), F_i += dvec * s, :459-480 */
    size_t Ek = 0;
    for (size_t gi = 0; gi < Gk; ++gi) Ek += (size_t)(b->edge_offset[graphs[gi] + 1] - b->edge_offset[graphs[gi]]);
    int* edges = xmalloc((Ek ? Ek : 1) * sizeof(int));
    Ek = 0;
    for (size_t gi = 0; gi < Gk; ++gi)
      for (int e = b->edge_offset[graphs[gi]]; e < b->edge_offset[graphs[gi] + 1]; ++e) edges[Ek++] = e;
    double* psi = xmalloc((Ek ? Ek : 1) * (H + 1) * sizeof(double));
    HO_PAR
    for (size_t ei = 0; ei < Ek; ++ei) {
      int e = edges[ei];
      const double* hd = h + (size_t)b->edge_dst[e] * H;
      const double* hs = h + (size_t)b->edge_src[e] * H;
      double* pe = psi + ei * (H + 1);
      for (size_t kk = 0; kk < H; ++kk) pe[kk] = hd[kk] + hs[kk];
      pe[H] = d[e];
    }
    double *fz[64], *fa[64];
    double* s = xmalloc((Ek ? Ek : 1) * sizeof(double));
    mlp_forward(hp, block, &HL, ff_first, psi, Ek, H + 1, fz, fa, s);
    for (size_t ei = 0; ei < Ek; ++ei) {
      int e = edges[ei];
      int i = b->edge_dst[e];
      for (int kk = 0; kk < 3; ++kk) forces[3 * (size_t)i + kk] += dvec[3 * (size_t)e + kk] * s[ei];
      if (c && c->s) c->s[e] = s[ei];
    }
    if (c && c->fz)
      for (int i = 0; i < D; ++i) {
        size_t od = HL.cols[ff_first + 2 * i];
        for (size_t ei = 0; ei < Ek; ++ei)
          for (size_t o = 0; o < od; ++o)
            c->fz[((size_t)i * E + edges[ei]) * W + o] = fz[i][ei * od + o];
      }
    for (int i = 0; i < D; ++i) free(fz[i]), free(fa[i]);
    free(s);
    free(psi);
    free(edges);
  }
  free(graphs);
  int rc = 0;
  for (size_t g = 0; g < G; ++g)
    if (!isfinite(energy[g])) rc = 6; /* :483-486 */
  for (size_t t = 0; t < 3 * N; ++t)
    if (!isfinite(forces[t])) rc = 6;
  free(d2), free(d), free(dvec), free(h), free(u), free(z1), free(a1), free(z2), free(m);
  free(agg), free(v), free(vz1), free(vp1), free(q);
  return rc;
}

/* ------------------------------------------------------------ backward ---- */
int ho_backward(const ho_hyper* hp, const double* shared, const double* const* heads,
                const ho_batch* b, const ho_cache* c, const double* d_energy,
                const double* d_forces, double* g_shared, double* const* g_heads) {
  if (!c || !c->h_in || !c->z1 || !c->a1 || !c->z2 || !c->agg || !c->vz1 || !c->vp1 ||
      !c->h_final || !c->ez || !c->fz)
    return 1; /* "model: missing forward cache", :495 */
  const size_t H = (size_t)hp->hidden, N = (size_t)b->N, E = (size_t)b->E, G = (size_t)b->G;
  const size_t W = (size_t)hp->head_width;
  const int D = hp->head_depth;
  lay_t SL, HL;
  lay_make(hp, 1, &SL);
  lay_make(hp, 0, &HL);
  const size_t PS = ho_shared_size(hp), PH = ho_head_size(hp);
  memset(g_shared, 0, PS * sizeof(double)); /* zero_grads, :189-194 */
  for (int k = 0; k < hp->n_heads; ++k)
    if (heads[k] && g_heads[k]) memset(g_heads[k], 0, PH * sizeof(double));

  double* d = xmalloc(E * sizeof(double));
  double* dvec = xmalloc(3 * E * sizeof(double));
  for (size_t e = 0; e < E; ++e) {
    const double* pi = b->pos + 3 * (size_t)b->edge_dst[e];
    const double* pj = b->pos + 3 * (size_t)b->edge_src[e];
    double dx = pi[0] - pj[0], dy = pi[1] - pj[1], dz = pi[2] - pj[2];
    if (b->edge_shift) dx -= b->edge_shift[3 * e], dy -= b->edge_shift[3 * e + 1], dz -= b->edge_shift[3 * e + 2];
    dvec[3 * e] = dx, dvec[3 * e + 1] = dy, dvec[3 * e + 2] = dz;
    d[e] = sqrt(dx * dx + dy * dy + dz * dz);
  }
  const double* h = c->h_final;
  double* dh = xmalloc(N * H * sizeof(double));
  int* graphs = xmalloc(G * sizeof(int));
  const int fe_first = 0, ff_first = 2 * D;

  for (int k = 0; k < hp->n_heads; ++k) {
    size_t Gk = 0;
    for (size_t g = 0; g < G; ++g)
      if (b->dataset_id[g] == k) graphs[Gk++] = (int)g;
    if (!Gk) continue;
    const double* block = heads[k];
    double* gblock = g_heads[k];
    /* energy branch, :512-524 -- rebuild the MLP cache (a_i = act(z_{i-1})) */
    double *ez[64], *ea[64];
    for (int i = 0; i < D; ++i) {
      size_t od = HL.cols[fe_first + 2 * i], in = HL.rows[fe_first + 2 * i];
      ez[i] = xmalloc(Gk * od * sizeof(double));
      ea[i] = xmalloc(Gk * in * sizeof(double));
      for (size_t gi = 0; gi < Gk; ++gi) {
        for (size_t o = 0; o < od; ++o) ez[i][gi * od + o] = c->ez[((size_t)i * G + graphs[gi]) * W + o];
        for (size_t t = 0; t < in; ++t) {
          if (i == 0) {
            /* pooled input: recompute exactly as forward */
            int g = graphs[gi];
            int lo = b->graph_offset[g], hi = b->graph_offset[g + 1];
            double acc = 0.0;
            for (int q = lo; q < hi; ++q) acc += h[(size_t)q * H + t];
            ea[i][gi * in + t] = acc * (1.0 / (double)(hi - lo));
          } else {
            ea[i][gi * in + t] = silu(c->ez[((size_t)(i - 1) * G + graphs[gi]) * W + t]);
          }
        }
      }
    }
    double* de = xmalloc(Gk * sizeof(double));
    for (size_t gi = 0; gi < Gk; ++gi) de[gi] = d_energy[graphs[gi]];
    double* dpooled = mlp_backward(hp, block, gblock, &HL, fe_first, Gk, ez, ea, de);
    for (size_t gi = 0; gi < Gk; ++gi) {
      int gr = graphs[gi];
      int lo = b->graph_offset[gr], hi = b->graph_offset[gr + 1];
      const double inv = 1.0 / (double)(hi - lo);
      for (int i = lo; i < hi; ++i)
        for (size_t kk = 0; kk < H; ++kk) dh[(size_t)i * H + kk] += dpooled[gi * H + kk] * inv;
    }
    for (int i = 0; i < D; ++i) free(ez[i]), free(ea[i]);
    free(de), free(dpooled);

    /* force branch, :526-549 */
    size_t Ek = 0;
    for (size_t gi = 0; gi < Gk; ++gi) Ek += (size_t)(b->edge_offset[graphs[gi] + 1] - b->edge_offset[graphs[gi]]);
    int* edges = xmalloc((Ek ? Ek : 1) * sizeof(int));
    Ek = 0;
    for (size_t gi = 0; gi < Gk; ++gi)
      for (int e = b->edge_offset[graphs[gi]]; e < b->edge_offset[graphs[gi] + 1]; ++e) edges[Ek++] = e;
    double *fz[64], *fa[64];
    for (int i = 0; i < D; ++i) {
      size_t od = HL.cols[ff_first + 2 * i], in = HL.rows[ff_first + 2 * i];
      fz[i] = xmalloc((Ek ? Ek : 1) * od * sizeof(double));
      fa[i] = xmalloc((Ek ? Ek : 1) * in * sizeof(double));
      HO_PAR
      for (size_t ei = 0; ei < Ek; ++ei) {
        int e = edges[ei];
        for (size_t o = 0; o < od; ++o) fz[i][ei * od + o] = c->fz[((size_t)i * E + e) * W + o];
        if (i == 0) {
          const double* hd = h + (size_t)b->edge_dst[e] * H;
          const double* hs = h + (size_t)b->edge_src[e] * H;
          for (size_t kk = 0; kk < H; ++kk) fa[i][ei * in + kk] = hd[kk] + hs[kk];
          fa[i][ei * in + H] = d[e];
        } else {
          for (size_t t = 0; t < in; ++t) fa[i][ei * in + t] = silu(c->fz[((size_t)(i - 1) * E + e) * W + t]);
        }
      }
    }
    double* ds = xmalloc((Ek ? Ek : 1) * sizeof(double));
    for (size_t ei = 0; ei < Ek; ++ei) {
      int e = edges[ei];
      int i = b->edge_dst[e];
      double acc = 0.0;
      for (int kk = 0; kk < 3; ++kk) acc += d_forces[3 * (size_t)i + kk] * dvec[3 * (size_t)e + kk];
      ds[ei] = acc;
    }
    double* dpsi = mlp_backward(hp, block, gblock, &HL, ff_first, Ek, fz, fa, ds);
    HO_PAR
    for (size_t k0 = 0; k0 < H; k0 += 4) { /* columns split; each in edge order */
      const size_t k1 = k0 + 4 < H ? k0 + 4 : H;
      for (size_t ei = 0; ei < Ek; ++ei) {
        int e = edges[ei];
        const double* dpe = dpsi + ei * (H + 1);
        double* dhd = dh + (size_t)b->edge_dst[e] * H;
        double* dhs = dh + (size_t)b->edge_src[e] * H;
        for (size_t kk = k0; kk < k1; ++kk) {
          dhd[kk] += dpe[kk];
          dhs[kk] += dpe[kk];
        }
      }
    }
    for (int i = 0; i < D; ++i) free(fz[i]), free(fa[i]);
    free(ds), free(dpsi), free(edges);
  }
  free(graphs);

  /* layers in reverse, :552-617 */
  const size_t K1 = 2 * H + 1;
  double* dvp1 = xmalloc(N * H * sizeof(double));
  double* dvz1 = xmalloc(N * H * sizeof(double));
  double* dv = xmalloc(N * 2 * H * sizeof(double));
  double* v = xmalloc(N * 2 * H * sizeof(double));
  double* dh_in = xmalloc(N * H * sizeof(double));
  double* dagg = xmalloc(N * H * sizeof(double));
  double* dz2 = xmalloc(E * H * sizeof(double));
  double* da1 = xmalloc(E * H * sizeof(double));
  double* du = xmalloc(E * K1 * sizeof(double));
  double* u = xmalloc(E * K1 * sizeof(double));
  double* d2 = xmalloc(E * sizeof(double));
  for (size_t e = 0; e < E; ++e) d2[e] = dvec[3 * e] * dvec[3 * e] + dvec[3 * e + 1] * dvec[3 * e + 1] + dvec[3 * e + 2] * dvec[3 * e + 2];
  for (int l = hp->layers - 1; l >= 0; --l) {
    const size_t base = 1 + 8 * (size_t)l;
    const double *eW1 = shared + SL.off[base + 0], *eW2 = shared + SL.off[base + 2];
    const double *nW1 = shared + SL.off[base + 4], *nW2 = shared + SL.off[base + 6];
    double *geW1 = g_shared + SL.off[base + 0], *geb1 = g_shared + SL.off[base + 1];
    double *geW2 = g_shared + SL.off[base + 2], *geb2 = g_shared + SL.off[base + 3];
    double *gnW1 = g_shared + SL.off[base + 4], *gnb1 = g_shared + SL.off[base + 5];
    double *gnW2 = g_shared + SL.off[base + 6], *gnb2 = g_shared + SL.off[base + 7];
    const double* hin = c->h_in + (size_t)l * N * H;
    const double* agg = c->agg + (size_t)l * N * H;
    const double* vz1 = c->vz1 + (size_t)l * N * H;
    const double* vp1 = c->vp1 + (size_t)l * N * H;
    const double* z1 = c->z1 + (size_t)l * E * H;
    const double* a1 = c->a1 + (size_t)l * E * H;
    const double* z2 = c->z2 + (size_t)l * E * H;
    /* node path, :569-587 */
    linear_backward(vp1, N, H, nW2, H, dh, gnW2, gnb2, dvp1);
    for (size_t t = 0; t < N * H; ++t) dvz1[t] = dvp1[t] * silu_grad(vz1[t]);
    for (size_t i = 0; i < N; ++i) {
      for (size_t k = 0; k < H; ++k) v[i * 2 * H + k] = hin[i * H + k];
      for (size_t k = 0; k < H; ++k) v[i * 2 * H + H + k] = agg[i * H + k];
    }
    linear_backward(v, N, 2 * H, nW1, H, dvz1, gnW1, gnb1, dv);
    memcpy(dh_in, dh, N * H * sizeof(double));
    for (size_t i = 0; i < N; ++i)
      for (size_t kk = 0; kk < H; ++kk) {
        dh_in[i * H + kk] += dv[i * 2 * H + kk];
        dagg[i * H + kk] = dv[i * 2 * H + H + kk];
      }
    /* edge path, :589-615 */
    HO_PAR
    for (size_t e = 0; e < E; ++e) {
      const double* da = dagg + (size_t)b->edge_dst[e] * H;
      for (size_t kk = 0; kk < H; ++kk) dz2[e * H + kk] = da[kk] * silu_grad(z2[e * H + kk]);
    }
    linear_backward(a1, E, H, eW2, H, dz2, geW2, geb2, da1);
    HO_PAR
    for (size_t t = 0; t < E * H; ++t) da1[t] = da1[t] * silu_grad(z1[t]);
    HO_PAR
    for (size_t e = 0; e < E; ++e) {
      double* ue = u + e * K1;
      const double* hd = hin + (size_t)b->edge_dst[e] * H;
      const double* hs = hin + (size_t)b->edge_src[e] * H;
      for (size_t k = 0; k < H; ++k) ue[k] = hd[k];
      for (size_t k = 0; k < H; ++k) ue[H + k] = hs[k];
      ue[2 * H] = d2[e];
    }
    linear_backward(u, E, K1, eW1, H, da1, geW1, geb1, du);
    HO_PAR
    for (size_t k0 = 0; k0 < H; k0 += 4) { /* columns split; each in edge order */
      const size_t k1 = k0 + 4 < H ? k0 + 4 : H;
      for (size_t e = 0; e < E; ++e) {
        const double* due = du + e * K1;
        double* dhd = dh_in + (size_t)b->edge_dst[e] * H;
        double* dhs = dh_in + (size_t)b->edge_src[e] * H;
        for (size_t kk = k0; kk < k1; ++kk) {
          dhd[kk] += due[kk];
          dhs[kk] += due[H + kk];
        }
      }
    }
    memcpy(dh, dh_in, N * H * sizeof(double));
  }
  /* embedding gradient, :619-622 */
  double* gembed = g_shared + SL.off[0];
  for (size_t i = 0; i < N; ++i)
    for (size_t kk = 0; kk < H; ++kk) gembed[(size_t)b->species[i] * H + kk] += dh[i * H + kk];
  free(d), free(dvec), free(dh), free(dvp1), free(dvz1), free(dv), free(v), free(dh_in);
  free(dagg), free(dz2), free(da1), free(du), free(u), free(d2);
  return 0;
}

/* ---------------------------------------------------------- trainer ------- */
/* per-graph w_E (E^-E)^2 + w_F mean_i ||F^_i - F_i||^2, mean over graphs */
double ho_loss(const ho_batch* b, const double* energy, const double* forces,
               const double* label_energy, const double* label_force, double w_e,
               double w_f, double* d_energy, double* d_forces) {
  const int G = b->G;
  double acc = 0.0;
  for (int g = 0; g < G; ++g) {
    const int lo = b->graph_offset[g], hi = b->graph_offset[g + 1];
    const double n = (double)(hi - lo);
    const double de = energy[g] - label_energy[g];
    double fe = 0.0;
    for (int i = lo; i < hi; ++i)
      for (int k = 0; k < 3; ++k) {
        const double r = forces[3 * (size_t)i + k] - label_force[3 * (size_t)i + k];
        fe += r * r;
        if (d_forces) d_forces[3 * (size_t)i + k] = 2.0 * w_f * r / (n * (double)G);
      }
    acc += w_e * de * de + w_f * fe / n;
    if (d_energy) d_energy[g] = 2.0 * w_e * de / (double)G;
  }
  return acc / (double)G;
}

void ho_adamw(double* p, const double* g, double* m, double* v, size_t n, long step,
              double lr, double beta1, double beta2, double eps, double wd) {
  const double bc1 = 1.0 - pow(beta1, (double)step);
  const double bc2 = 1.0 - pow(beta2, (double)step);
  const double step_size = lr / bc1;
  const double bc2_sqrt = sqrt(bc2);
  for (size_t i = 0; i < n; ++i) {
    p[i] *= 1.0 - lr * wd;
    m[i] = beta1 * m[i] + (1.0 - beta1) * g[i];
    v[i] = beta2 * v[i] + (1.0 - beta2) * g[i] * g[i];
    const double denom = sqrt(v[i]) / bc2_sqrt + eps;
    p[i] -= step_size * m[i] / denom;
  }
}

// Internal host-side declarations shared by the translation units.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <vector>

#include "uc_common.cuh"

namespace uc {

// Per-level physics constants, derived on the host exactly as the numba
// prologues derive them (free_growth.py:97-108, alloy.py:137-147).
struct LevelConsts {
  double base, four_eps, eps32, reg, avg, avg_reg;
  double inv_dt_s;  // mass_sign / dt
  // free growth
  double well_c, drive_c, wbg, half_w, walpha, tmelt, latent;
  // alloy
  double weight, inv_dt, coupling, omk, half_k, half_omk, dq_c, at_coef, at_reg2, g4_coef,
      g4_shift;
  int normalized;
};

LevelConsts make_level(const uc_model_params& p, int dim, const uc_scheme& sc, bool new_level);
void make_jxw(const Grid& g, double* jxw);  // 9 or 27 entries, mesh.py:52-61,174-176

struct Precond;  // precond.cu

}  // namespace uc

// Reduction geometry: fixed so the summation tree depends on n only.
#define UC_RED_THREADS 256
#define UC_RED_GRID_MAX 1184
#define UC_MDOT_B 8  // dots per k_mdot launch (blas.cu); partials hold UC_MDOT_B x UC_RED_GRID_MAX
#define UC_SCAL_SLOTS 2048

struct uc_ctx {
  uc::Grid grid;
  uc_mesh_desc mesh;
  uc_model_params params;
  cudaStream_t stream = nullptr;
  int device = 0;
  int num_sms = 148;
  // reduction workspace
  double* partials = nullptr;    // [UC_MDOT_B * UC_RED_GRID_MAX]
  unsigned int* ticket = nullptr;
  double* scal = nullptr;        // [scal_cap] device scalars (grown on demand by the Arnoldi step)
  double* pinned = nullptr;      // [scal_cap] pinned host staging
  int scal_cap = UC_SCAL_SLOTS;
  unsigned int* flags = nullptr;      // [4] sticky status flags (device alias)
  unsigned int* flags_host = nullptr; // mapped pinned host memory
  unsigned long long* locate_key = nullptr;
  double* diag_ws = nullptr;      // diag.cu partials + ticket (lazy)
  double* ebuf = nullptr;         // residual.cu: edge contributions of the ring-free 2D tiles (lazy)
  size_t ebuf_n = 0;
  // ghost planes [slot][side] -> [2][plane]; slots 0 u, 1 old, 2 prev, 3 v, 4 state
  double* ghost[5][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr},
                         {nullptr, nullptr}, {nullptr, nullptr}};
  uc::Precond* pc = nullptr;
  // slab neighbours: a local context (same process/device) or a remote NCCL rank
  uc_ctx* lo_local = nullptr;
  uc_ctx* hi_local = nullptr;
  int lo_rank = -1, hi_rank = -1;
  bool dist = false;  // member of a multi-rank NCCL communicator
};

namespace uc {
typedef std::vector<uc_ctx*> Group;

// Addresses of the boundary / ghost planes of one logical vector per slab.
struct PlaneAddr {
  int nblocks = 2;
  std::function<int64_t(uc_ctx*)> count;
  std::function<const double*(uc_ctx*, int)> top, bottom;
  std::function<double*(uc_ctx*, int)> glo, ghi;
  // owned planes [slo, shi) of this vector's level; plane_ok filters which
  // boundary planes move (by global plane index); unset = all
  std::function<int64_t(uc_ctx*)> slo, shi;
  std::function<bool(int64_t)> plane_ok;
};
// comm.cu
bool group_has_remote(const Group& g);
bool comm_is_host();  // remote neighbours go through the host-staged transport
void comm_rank_world(int& rank, int& world);  // this process's rank and the number of ranks (0, 1 without a communicator)
int exchange(const Group& g, const PlaneAddr& addr, bool dir_up, bool dir_down, cudaStream_t s);
int global_sum(const Group& g, double* const* slots, bool do_sqrt, cudaStream_t s);
int global_sum_n(const Group& g, double* const* slots, int n, cudaStream_t s);
bool group_needs_sum(const Group& g);
// exchange ghost planes of unpadded block vectors vecs[i] into ghost slot `slot`
int halo_vectors(const Group& g, int slot, const double* const* vecs, cudaStream_t s);
// blas.cu
int reduce_dot(uc_ctx* c, int64_t n, const double* a, const double* b, double* out_dev,
               bool sqrt_result);
int nonfinite_flag(uc_ctx* c, int64_t n, const double* a, unsigned int* flag);
int nonfinite_flag_on(cudaStream_t s, int64_t n, const double* a, unsigned int* flag);
int launch_axpy(uc_ctx* c, int64_t n, const double* a, double s, const double* b, double* out);
// grow the scalar workspace to at least `need` slots (synchronises the stream when it grows)
int ensure_scal(uc_ctx* c, int64_t need);
// residual.cu
enum { MODE_NEW = 0, MODE_OLD = 1, MODE_JV = 2 };
int launch_residual(uc_ctx* c, const uc_scheme* sc, int mode, const double* u,
                    const double* old, const double* prev, const double* v, const double* fu,
                    const double* fixed, double* out, double eps_num, const double* vnorm_dev,
                    double* eps_out);
int locate_nonfinite(uc_ctx* c, const uc_scheme* sc, int part, const double* u,
                     const double* old, const double* prev, int64_t out[5],
                     const uint8_t* emask = nullptr);
int launch_subset(uc_ctx* c, const uc_scheme* sc, int mode, const double* u, const double* old,
                  const double* prev, const double* fixed, const uint8_t* emask, double* out);
void make_jxw(const Grid& g, double* jxw);
// massdiff.cu (single-field test model)
int launch_massdiff(uc_ctx* c, const uc_scheme* sc, int mode, const double* u, const double* old,
                    const double* v, const double* fu, const double* fixed, double* out,
                    double eps_num, const double* vnorm_dev, double* eps_out);
int launch_massdiff_subset(uc_ctx* c, const uc_scheme* sc, int mode, const double* u,
                           const double* old, const double* fixed, const uint8_t* emask, double* out);
int locate_massdiff(uc_ctx* c, const uc_scheme* sc, int mode, const double* u, const double* old,
                    const uint8_t* emask, unsigned long long* key_dev);
// entries per vector: fields x owned nodes
inline int64_t vec_len(const uc_ctx* c) {
  return (c->params.model == UC_MODEL_MASS_DIFF ? 1 : 2) * c->grid.nloc;
}
// precond.cu
int precond_build(uc_ctx* c, const uc_scheme* sc, const double* state, const uc_precond_cfg* cfg);
int precond_build_group(const Group& G, const uc_scheme* sc, const double* const* states,
                        const uc_precond_cfg* cfg);
int precond_apply_group(const Group& G, const double* const* v, double* const* out);
int precond_apply(uc_ctx* c, const double* v, double* out);
int precond_stencil(uc_ctx* c, int level, int block, double* host_out);
int precond_levels(uc_ctx* c, int64_t* shapes);
int precond_uniform_fraction(uc_ctx* c, int level, int block, double* frac);
void precond_destroy(Precond* p);
}  // namespace uc

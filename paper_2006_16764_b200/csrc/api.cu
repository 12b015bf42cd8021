// C ABI entry points: context management, residual / Jv, status.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "uc_internal.h"

namespace uc {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int set_cuda_error(cudaError_t e, const char* what, const char* file, int line) {
  return set_error(UC_ERR_CUDA, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
}

static int build_grid(const uc_mesh_desc* m, Grid* g) {
  if (m->dim != 2 && m->dim != 3) return set_error(UC_ERR_ARG, "dimension must be 2 or 3");
  if (m->order != 1)
    return set_error(UC_ERR_UNSUPPORTED, "only Q1 elements run on the device (order=%d)", m->order);
  memset(g, 0, sizeof(*g));
  g->dim = m->dim;
  for (int a = 0; a < 3; ++a) {
    if (a < m->dim) {
      if (m->counts[a] < 1) return set_error(UC_ERR_ARG, "element counts must be at least 1");
      if (!(m->spacing[a] > 0.0)) return set_error(UC_ERR_ARG, "spacing must be positive");
      g->ne[a] = m->counts[a];
      g->nn[a] = m->counts[a] + 1;
      g->h[a] = m->spacing[a];
      g->ih[a] = 0.5 * (2.0 / m->spacing[a]);
    } else {
      g->ne[a] = 1;
      g->nn[a] = 1;
      g->h[a] = 1.0;
      g->ih[a] = 1.0;
    }
  }
  const int s = m->dim - 1;
  g->nslow = g->nn[s];
  g->eslow = g->ne[s];
  g->plane = m->dim == 3 ? g->nn[0] * g->nn[1] : g->nn[0];
  g->lo = m->slab_lo;
  g->hi = m->slab_hi;
  if (g->lo < 0 || g->hi > g->nslow || g->lo >= g->hi)
    return set_error(UC_ERR_ARG, "bad slab [%lld, %lld) of %lld planes", (long long)g->lo,
                     (long long)g->hi, (long long)g->nslow);
  g->nloc = (g->hi - g->lo) * g->plane;
  return UC_OK;
}

}  // namespace uc

using namespace uc;

extern "C" {

int uc_abi_version(void) { return 1; }

const char* uc_last_error(void) { return g_err; }

int uc_ctx_create(const uc_mesh_desc* mesh, const uc_model_params* params, void* stream,
                  uc_ctx** out) {
  if (!mesh || !params || !out) return set_error(UC_ERR_ARG, "uc_ctx_create: NULL argument");
  if (params->model != UC_MODEL_FREE_GROWTH && params->model != UC_MODEL_ALLOY &&
      params->model != UC_MODEL_MASS_DIFF)
    return set_error(UC_ERR_UNSUPPORTED, "unknown model %d", params->model);
  if (params->model == UC_MODEL_MASS_DIFF &&
      (mesh->slab_lo != 0 || mesh->slab_hi != mesh->counts[mesh->dim > 0 ? mesh->dim - 1 : 0] + 1))
    return set_error(UC_ERR_UNSUPPORTED, "the mass-diffusion test model runs on a single slab only");
  uc_ctx* c = new uc_ctx();
  int rc = build_grid(mesh, &c->grid);
  if (rc) {
    delete c;
    return rc;
  }
  c->mesh = *mesh;
  c->params = *params;
  c->stream = (cudaStream_t)stream;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
  if (e == cudaSuccess) e = cudaMalloc(&c->partials, sizeof(double) * UC_MDOT_B * UC_RED_GRID_MAX);
  if (e == cudaSuccess) e = cudaMalloc(&c->ticket, sizeof(unsigned int) * 4);
  if (e == cudaSuccess) e = cudaMemset(c->ticket, 0, sizeof(unsigned int) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&c->scal, sizeof(double) * UC_SCAL_SLOTS);
  if (e == cudaSuccess) e = cudaMemset(c->scal, 0, sizeof(double) * UC_SCAL_SLOTS);
  if (e == cudaSuccess) e = cudaMallocHost(&c->pinned, sizeof(double) * UC_SCAL_SLOTS);
  // status flags live in mapped pinned host memory: kernels set them, the
  // host reads them after a stream sync without a device->host copy
  if (e == cudaSuccess) e = cudaHostAlloc(&c->flags_host, sizeof(unsigned int) * 4, cudaHostAllocMapped);
  if (e == cudaSuccess) {
    memset(c->flags_host, 0, sizeof(unsigned int) * 4);
    e = cudaHostGetDevicePointer(&c->flags, c->flags_host, 0);
  }
  if (e == cudaSuccess) e = cudaMalloc(&c->locate_key, sizeof(unsigned long long));
  const Grid& g = c->grid;
  if (e == cudaSuccess && g.lo > 0) {
    for (int s = 0; s < 5 && e == cudaSuccess; ++s) e = cudaMalloc(&c->ghost[s][0], sizeof(double) * 2 * g.plane);
  }
  if (e == cudaSuccess && g.hi < g.nslow) {
    for (int s = 0; s < 5 && e == cudaSuccess; ++s) e = cudaMalloc(&c->ghost[s][1], sizeof(double) * 2 * g.plane);
  }
  if (e != cudaSuccess) {
    rc = set_cuda_error(e, "uc_ctx_create allocation", __FILE__, __LINE__);
    uc_ctx_destroy(c);
    return rc;
  }
  *out = c;
  return UC_OK;
}

int uc_ctx_destroy(uc_ctx* c) {
  if (!c) return UC_OK;
  if (c->pc) precond_destroy(c->pc);
  cudaFree(c->partials);
  cudaFree(c->ticket);
  cudaFree(c->scal);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->flags_host) cudaFreeHost(c->flags_host);
  cudaFree(c->locate_key);
  cudaFree(c->diag_ws);
  cudaFree(c->ebuf);
  for (int s = 0; s < 5; ++s)
    for (int d = 0; d < 2; ++d) cudaFree(c->ghost[s][d]);
  delete c;
  return UC_OK;
}

int uc_set_stream(uc_ctx* c, void* stream) {
  if (!c) return set_error(UC_ERR_ARG, "NULL context");
  c->stream = (cudaStream_t)stream;
  return UC_OK;
}

int64_t uc_n_local(const uc_ctx* c) { return c ? c->grid.nloc : -1; }

double* uc_ghost_ptr(uc_ctx* c, int slot, int side) {
  if (!c || slot < 0 || slot > 4 || side < 0 || side > 1) return nullptr;
  return c->ghost[slot][side];
}

int uc_residual_group(uc_ctx* const* ctxs, int n, const uc_scheme* sc, int part,
                      const double* const* unew, const double* const* old,
                      const double* const* prev, const double* const* fixed, double* const* out) {
  if (!ctxs || n < 1 || !sc || !old || !prev || !out)
    return set_error(UC_ERR_ARG, "uc_residual: NULL argument");
  if (!(sc->dt > 0.0) || sc->theta < 0.0 || sc->theta > 1.0)
    return set_error(UC_ERR_ARG, "uc_residual: bad scheme");
  if (part != UC_PART_OLD && (part != UC_PART_NEW || !unew || !fixed))
    return set_error(UC_ERR_ARG, "uc_residual: bad part");
  Group G(ctxs, ctxs + n);
  cudaStream_t s = G[0]->stream;
  int rc;
  if ((rc = halo_vectors(G, 1, old, s))) return rc;
  if ((rc = halo_vectors(G, 2, prev, s))) return rc;
  if (part == UC_PART_NEW && (rc = halo_vectors(G, 0, unew, s))) return rc;
  for (int i = 0; i < n; ++i) {
    if (part == UC_PART_OLD)
      rc = launch_residual(G[i], sc, MODE_OLD, nullptr, old[i], prev[i], nullptr, nullptr, nullptr,
                           out[i], 0.0, nullptr, nullptr);
    else
      rc = launch_residual(G[i], sc, MODE_NEW, unew[i], old[i], prev[i], nullptr, nullptr, fixed[i],
                           out[i], 0.0, nullptr, nullptr);
    if (rc) return rc;
  }
  return UC_OK;
}

int uc_residual(uc_ctx* c, const uc_scheme* sc, int part, const double* unew, const double* old,
                const double* prev, const double* fixed, double* out) {
  return uc_residual_group(&c, 1, sc, part, &unew, &old, &prev, &fixed, &out);
}

int uc_residual_subset(uc_ctx* c, const uc_scheme* sc, int part, const double* unew,
                       const double* old, const double* prev, const double* fixed,
                       const uint8_t* element_mask, double* out) {
  if (!c || !sc || !old || !prev || !element_mask || !out)
    return set_error(UC_ERR_ARG, "uc_residual_subset: NULL argument");
  if (!(sc->dt > 0.0)) return set_error(UC_ERR_ARG, "uc_residual_subset: bad scheme");
  if (part != UC_PART_OLD && (part != UC_PART_NEW || !unew))
    return set_error(UC_ERR_ARG, "uc_residual_subset: bad part");
  if (c->grid.lo != 0 || c->grid.hi != c->grid.nslow)
    return set_error(UC_ERR_UNSUPPORTED, "element subsets are assembled on a single slab only");
  return launch_subset(c, sc, part == UC_PART_OLD ? MODE_OLD : MODE_NEW, unew, old, prev, fixed,
                       element_mask, out);
}

int uc_locate_nonfinite_subset(uc_ctx* c, const uc_scheme* sc, int part, const double* unew,
                               const double* old, const double* prev, const uint8_t* element_mask,
                               int64_t* field, int64_t* which, int64_t* element, int64_t* qp,
                               int64_t* first_node) {
  if (!c || !sc) return set_error(UC_ERR_ARG, "uc_locate_nonfinite: NULL argument");
  int64_t o[5];
  int rc = locate_nonfinite(c, sc, part, unew, old, prev, o, element_mask);
  if (rc < 0 || rc > 1) return rc;
  *field = o[0];
  *which = o[1];
  *element = o[2];
  *qp = o[3];
  *first_node = o[4];
  return UC_OK;
}

int uc_locate_nonfinite(uc_ctx* c, const uc_scheme* sc, int part, const double* unew,
                        const double* old, const double* prev, int64_t* field, int64_t* which,
                        int64_t* element, int64_t* qp, int64_t* first_node) {
  if (!c || !sc) return set_error(UC_ERR_ARG, "uc_locate_nonfinite: NULL argument");
  int64_t o[5];
  int rc = locate_nonfinite(c, sc, part, unew, old, prev, o);
  if (rc < 0 || rc > 1) return rc;
  *field = o[0];
  *which = o[1];
  *element = o[2];
  *qp = o[3];
  *first_node = o[4];
  return UC_OK;
}

int uc_jv_group(uc_ctx* const* ctxs, int n, const uc_scheme* sc, const double* const* u,
                const double* const* fu, const double* const* v, double unorm,
                const double* const* old, const double* const* prev, const double* const* fixed,
                double* const* jv, double* eps_out) {
  if (!ctxs || n < 1 || !sc || !u || !fu || !v || !old || !prev || !fixed || !jv)
    return set_error(UC_ERR_ARG, "uc_jv: NULL argument");
  Group G(ctxs, ctxs + n);
  cudaStream_t s = G[0]->stream;
  int rc;
  if ((rc = halo_vectors(G, 1, old, s))) return rc;
  if ((rc = halo_vectors(G, 2, prev, s))) return rc;
  if ((rc = halo_vectors(G, 0, u, s))) return rc;
  if ((rc = halo_vectors(G, 3, v, s))) return rc;
  // |v| on the device (newton.py:108), then eps = EPS0*sqrt(1+|u|)/|v| in-kernel
  std::vector<double*> vn(n);
  const bool sum = group_needs_sum(G);
  for (int i = 0; i < n; ++i) {
    vn[i] = G[i]->scal + (G[i]->scal_cap - 1);
    if ((rc = reduce_dot(G[i], vec_len(G[i]), v[i], nullptr, vn[i], !sum))) return rc;
  }
  if (sum && (rc = global_sum(G, vn.data(), true, s))) return rc;
  const double eps_num = UC_EPS0 * sqrt(1.0 + unorm);
  for (int i = 0; i < n; ++i)
    if ((rc = launch_residual(G[i], sc, MODE_JV, u[i], old[i], prev[i], v[i], fu[i], fixed[i], jv[i],
                              eps_num, vn[i], i == 0 ? eps_out : nullptr)))
      return rc;
  return UC_OK;
}

int uc_jv(uc_ctx* c, const uc_scheme* sc, const double* u, const double* fu, const double* v,
          double unorm, const double* old, const double* prev, const double* fixed, double* jv,
          double* eps_out) {
  return uc_jv_group(&c, 1, sc, &u, &fu, &v, unorm, &old, &prev, &fixed, &jv, eps_out);
}

int uc_dot_group(uc_ctx* const* ctxs, int n, const double* const* a, const double* const* b,
                 int do_sqrt, double* out) {
  if (!ctxs || n < 1 || !a || !out) return set_error(UC_ERR_ARG, "uc_dot_group: NULL argument");
  Group G(ctxs, ctxs + n);
  cudaStream_t s = G[0]->stream;
  std::vector<double*> slot(n);
  int rc;
  for (int i = 0; i < n; ++i) {
    slot[i] = G[i]->scal + (G[i]->scal_cap - 2);
    if ((rc = reduce_dot(G[i], vec_len(G[i]), a[i], b ? b[i] : nullptr, slot[i], false))) return rc;
  }
  if ((rc = global_sum(G, slot.data(), do_sqrt != 0, s))) return rc;
  UC_CUDA_OK(cudaMemcpyAsync(G[0]->pinned, slot[0], sizeof(double), cudaMemcpyDeviceToHost, s));
  UC_CUDA_OK(cudaStreamSynchronize(s));
  *out = G[0]->pinned[0];
  return UC_OK;
}

int uc_precond_build_group(uc_ctx* const* ctxs, int n, const uc_scheme* sc,
                           const double* const* states, const uc_precond_cfg* cfg) {
  if (!ctxs || n < 1 || !sc || !states || !cfg) return set_error(UC_ERR_ARG, "uc_precond_build: NULL argument");
  if (ctxs[0]->params.model == UC_MODEL_MASS_DIFF)
    return set_error(UC_ERR_UNSUPPORTED, "the mass-diffusion test model has no preconditioner coefficients");
  Group G(ctxs, ctxs + n);
  return precond_build_group(G, sc, states, cfg);
}

int uc_precond_apply_group(uc_ctx* const* ctxs, int n, const double* const* v, double* const* out) {
  if (!ctxs || n < 1 || !v || !out) return set_error(UC_ERR_ARG, "uc_precond_apply: NULL argument");
  Group G(ctxs, ctxs + n);
  return precond_apply_group(G, v, out);
}

int uc_status(uc_ctx* c, uc_status_t* out, int clear) {
  if (!c || !out) return set_error(UC_ERR_ARG, "uc_status: NULL argument");
  UC_CUDA_OK(cudaStreamSynchronize(c->stream));
  volatile unsigned int* f = c->flags_host;
  out->residual_nonfinite = (int)f[0];
  out->precond_nonfinite = (int)f[1];
  out->precond_bad_diag = (int)f[2];
  out->pad = 0;
  if (clear) {
    f[0] = 0u;
    f[1] = 0u;
    f[2] = 0u;
  }
  return UC_OK;
}

int uc_precond_build(uc_ctx* c, const uc_scheme* sc, const double* state, const uc_precond_cfg* cfg) {
  if (!c || !sc || !state || !cfg) return set_error(UC_ERR_ARG, "uc_precond_build: NULL argument");
  return precond_build(c, sc, state, cfg);
}

int uc_precond_apply(uc_ctx* c, const double* v, double* out) {
  if (!c || !v || !out) return set_error(UC_ERR_ARG, "uc_precond_apply: NULL argument");
  return precond_apply(c, v, out);
}

int uc_precond_stencil(uc_ctx* c, int level, int block, double* host_out) {
  if (!c || !host_out) return set_error(UC_ERR_ARG, "uc_precond_stencil: NULL argument");
  return precond_stencil(c, level, block, host_out);
}

int uc_precond_uniform(uc_ctx* c, int level, int block, double* frac) {
  if (!c || !frac) return set_error(UC_ERR_ARG, "uc_precond_uniform: NULL argument");
  return precond_uniform_fraction(c, level, block, frac);
}

int uc_precond_levels(uc_ctx* c, int64_t* shapes) {
  if (!c) return set_error(UC_ERR_ARG, "uc_precond_levels: NULL argument");
  return precond_levels(c, shapes);
}

}  // extern "C"

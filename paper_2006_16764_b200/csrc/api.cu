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
  if (params->model != UC_MODEL_FREE_GROWTH && params->model != UC_MODEL_ALLOY)
    return set_error(UC_ERR_UNSUPPORTED, "unknown model %d", params->model);
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
  if (e == cudaSuccess) e = cudaMalloc(&c->partials, sizeof(double) * UC_RED_GRID_MAX);
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
    for (int s = 0; s < 4 && e == cudaSuccess; ++s) e = cudaMalloc(&c->ghost[s][0], sizeof(double) * 2 * g.plane);
  }
  if (e == cudaSuccess && g.hi < g.nslow) {
    for (int s = 0; s < 4 && e == cudaSuccess; ++s) e = cudaMalloc(&c->ghost[s][1], sizeof(double) * 2 * g.plane);
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
  for (int s = 0; s < 4; ++s)
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
  if (!c || slot < 0 || slot > 3 || side < 0 || side > 1) return nullptr;
  return c->ghost[slot][side];
}

int uc_residual(uc_ctx* c, const uc_scheme* sc, int part, const double* unew, const double* old,
                const double* prev, const double* fixed, double* out) {
  if (!c || !sc || !old || !prev || !out) return set_error(UC_ERR_ARG, "uc_residual: NULL argument");
  if (!(sc->dt > 0.0) || sc->theta < 0.0 || sc->theta > 1.0)
    return set_error(UC_ERR_ARG, "uc_residual: bad scheme");
  if (part == UC_PART_OLD)
    return launch_residual(c, sc, MODE_OLD, nullptr, old, prev, nullptr, nullptr, nullptr, out,
                           0.0, nullptr, nullptr);
  if (part != UC_PART_NEW || !unew || !fixed) return set_error(UC_ERR_ARG, "uc_residual: bad part");
  return launch_residual(c, sc, MODE_NEW, unew, old, prev, nullptr, nullptr, fixed, out, 0.0,
                         nullptr, nullptr);
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

int uc_jv(uc_ctx* c, const uc_scheme* sc, const double* u, const double* fu, const double* v,
          double unorm, const double* old, const double* prev, const double* fixed, double* jv,
          double* eps_out) {
  if (!c || !sc || !u || !fu || !v || !old || !prev || !fixed || !jv)
    return set_error(UC_ERR_ARG, "uc_jv: NULL argument");
  // |v| on the device (newton.py:108), then eps = EPS0*sqrt(1+|u|)/|v| in-kernel
  double* vnorm = c->scal + (UC_SCAL_SLOTS - 1);
  int rc = reduce_dot(c, 2 * c->grid.nloc, v, nullptr, vnorm, true);
  if (rc) return rc;
  const double eps_num = UC_EPS0 * sqrt(1.0 + unorm);
  return launch_residual(c, sc, MODE_JV, u, old, prev, v, fu, fixed, jv, eps_num, vnorm, eps_out);
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

int uc_precond_levels(uc_ctx* c, int64_t* shapes) {
  if (!c) return set_error(UC_ERR_ARG, "uc_precond_levels: NULL argument");
  return precond_levels(c, shapes);
}

}  // extern "C"

// Per-step diagnostics of the time loop, on the device.
//
// Replaces the host passes the reference's simulate() makes over the new state
// after every converged step (undercool/driver.py:186-229):
//   blow-up test      np.isfinite(u_new).all(), np.max(np.abs(u_new))  (:186-188)
//   _heat_balance     w @ (T_new - T_old), w @ (phi_new - phi_old),
//                     w @ (phi_old - phi_prev) with the nodal integration
//                     weights w = mesh.integration_weights() (:86-98,
//                     mesh.py:130-143)
//   _total_solute     sum over elements of c(u, phi) @ jxw at the new level
//                     (:76-83, alloy.py:119-127)
//   extract_tip       last crossing of phi through the contour level along the
//                     first node row, linear interpolation (diagnostics.py:69-89)
// One pass per quantity family; each CTA reduces in registers + warp shuffles
// and the last CTA (ticket) folds the per-CTA partials in index order, so the
// results are bitwise reproducible.  A context reports over its owned slab;
// the host combines slabs (sums in slab order, max, the tip from plane 0).
#include "uc_internal.h"

namespace uc {

enum { D_NONFINITE = 0, D_MAXABS, D_ST, D_SPN, D_SPO, D_SOLUTE, D_TIP, D_FOUND };
#define UC_DIAG_THREADS 256
#define UC_DIAG_GRID_MAX 592

struct DiagArgs {
  Grid g;
  const double* nw;  // new state, owned block vector [2][nloc]
  const double* od;  // old state
  const double* pv;  // prev state (field 0 used)
  const double* ghi; // plane hi of the new state (slab runs), NULL otherwise
  double enw[8];     // jxw @ values per local node (mesh.py:136)
  double jxw[27];
  double comp_over_2k, kpart;
  double level, extent_x;
  double* ws;        // [6][UC_DIAG_GRID_MAX] partials
  unsigned int* ticket;
  double* out;
};

__device__ __forceinline__ double bsum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
  return s;  // thread 0
}
__device__ __forceinline__ double bmax(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = fmax(s, sh[w]);
  return s;
}

// nodal integration weight of global node (i, j, k): bincount of the
// per-element weights in element-id order (mesh.py:137-141)
__device__ __forceinline__ double node_weight(const DiagArgs& a, int64_t i, int64_t j, int64_t k) {
  const Grid& g = a.g;
  double w = 0.0;
  const int cmax = g.dim == 3 ? 1 : 0;
  for (int c = cmax; c >= 0; --c)
    for (int b = 1; b >= 0; --b)
      for (int aa = 1; aa >= 0; --aa) {
        const int64_t ex = i - aa, ey = j - b, ez = k - c;
        if (ex < 0 || ex >= g.ne[0] || ey < 0 || ey >= g.ne[1]) continue;
        if (g.dim == 3 && (ez < 0 || ez >= g.ne[2])) continue;
        w += a.enw[aa + 2 * b + 4 * c];
      }
  return w;
}

// Finish: thread 0 of each CTA holds `nv` values; the last CTA folds them in
// CTA order into out[first..first+nv).  kinds: 0 sum, 1 max.
template <int NV>
__device__ void finish(const DiagArgs& a, const double (&v)[NV], const int (&kind)[NV], int first,
                       double* sh) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    for (int j = 0; j < NV; ++j) a.ws[j * UC_DIAG_GRID_MAX + blockIdx.x] = v[j];
    __threadfence();
    last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int j = 0; j < NV; ++j) {
    double x = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
      const double p = __ldcg(a.ws + j * UC_DIAG_GRID_MAX + b);
      x = kind[j] ? fmax(x, p) : x + p;
    }
    const double t = kind[j] ? bmax(x, sh) : bsum(x, sh);
    if (threadIdx.x == 0) a.out[first + j] = t;
  }
  if (threadIdx.x == 0) *a.ticket = 0u;
}

__global__ void __launch_bounds__(UC_DIAG_THREADS) k_diag_nodes(const DiagArgs a, int balance) {
  __shared__ double sh[32];
  const Grid& g = a.g;
  double bad = 0.0, mx = 0.0, st = 0.0, spn = 0.0, spo = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.nloc; q += stride) {
    const double p1 = a.nw[q], t1 = a.nw[g.nloc + q];
    if (!isfinite(p1)) bad += 1.0;
    if (!isfinite(t1)) bad += 1.0;
    mx = fmax(mx, fmax(fabs(p1), fabs(t1)));
    if (balance) {
      const int64_t gid = g.lo * g.plane + q;
      const int64_t i = gid % g.nn[0], r = gid / g.nn[0];
      const int64_t j = g.dim == 3 ? r % g.nn[1] : r, k = g.dim == 3 ? r / g.nn[1] : 0;
      const double w = node_weight(a, i, j, k);
      const double p0 = a.od[q], t0 = a.od[g.nloc + q], pp = a.pv[q];
      st = fma(w, __dsub_rn(t1, t0), st);
      spn = fma(w, __dsub_rn(p1, p0), spn);
      spo = fma(w, __dsub_rn(p0, pp), spo);
    }
  }
  double v[5];
  v[0] = bsum(bad, sh);
  v[1] = bmax(mx, sh);
  v[2] = bsum(st, sh);
  v[3] = bsum(spn, sh);
  v[4] = bsum(spo, sh);
  const int kind[5] = {0, 1, 0, 0, 0};
  finish<5>(a, v, kind, D_NONFINITE, sh);
}

// composition integral over the owned element layers [lo, min(hi, eslow))
template <int DIM>
__global__ void __launch_bounds__(UC_DIAG_THREADS) k_diag_solute(const DiagArgs a) {
  __shared__ double sh[32];
  const Grid& g = a.g;
  constexpr int NL = DIM == 3 ? 8 : 4, NQ = DIM == 3 ? 27 : 9;
  const int64_t lay_end = g.hi < g.eslow ? g.hi : g.eslow;
  const int64_t lat_e = g.ne[0] * (DIM == 3 ? g.ne[1] : 1);
  const int64_t ne = (lay_end - g.lo) * lat_e;
  const double omk = 1.0 - a.kpart, opk = 1.0 + a.kpart;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += stride) {
    const int64_t lay = g.lo + e / lat_e, le = e % lat_e;
    const int64_t ex = le % g.ne[0], ey = DIM == 3 ? le / g.ne[0] : 0;
    double ph[NL], uu[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int jx = l & 1, jy = (l >> 1) & 1, jz = l >> 2;
      const int64_t p = lay + (DIM == 3 ? jz : jy);
      const int64_t lat = (ex + jx) + (DIM == 3 ? (ey + jy) * g.nn[0] : 0);
      if (p < g.hi) {
        const int64_t idx = (p - g.lo) * g.plane + lat;
        ph[l] = a.nw[idx];
        uu[l] = a.nw[g.nloc + idx];
      } else {
        ph[l] = a.ghi[lat];
        uu[l] = a.ghi[g.plane + lat];
      }
    }
    double es = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int qx = q % 3, qy = (q / 3) % 3, qz = q / 9;
      double fq = 0.0, uq = 0.0;
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int jx = l & 1, jy = (l >> 1) & 1, jz = l >> 2;
        // basis value as mesh.py:163-167 rounds it: (1*Lx)*Ly(*Lz)
        double bv = lq(jx, qx) * lq(jy, qy);
        if (DIM == 3) bv = bv * lq(jz, qz);
        fq = fma(bv, ph[l], fq);
        uq = fma(bv, uu[l], uq);
      }
      // map_u_to_c (alloy.py:119-127), numpy operation order
      const double c = __dmul_rn(__dmul_rn(a.comp_over_2k, __dsub_rn(opk, __dmul_rn(omk, fq))),
                                 __dadd_rn(1.0, __dmul_rn(omk, uq)));
      es = fma(c, a.jxw[q], es);
    }
    acc += es;
  }
  double v[1];
  v[0] = bsum(acc, sh);
  const int kind[1] = {0};
  finish<1>(a, v, kind, D_SOLUTE, sh);
}

// extract_tip along the first node row (needs plane 0: the slab with lo == 0)
__global__ void __launch_bounds__(1024) k_diag_tip(const DiagArgs a) {
  __shared__ long long s_cross, s_exact;
  const Grid& g = a.g;
  const int64_t nx = g.nn[0];
  if (threadIdx.x == 0) {
    s_cross = -1;
    s_exact = -1;
  }
  __syncthreads();
  long long cross = -1, exact = -1;
  for (int64_t i = threadIdx.x; i < nx; i += blockDim.x) {
    const double d = __dsub_rn(a.nw[i], a.level);
    if (d == 0.0) exact = i;
    if (i + 1 < nx) {
      const double d1 = __dsub_rn(a.nw[i + 1], a.level);
      if (__dmul_rn(d, d1) < 0.0) cross = i;
    }
  }
  atomicMax(&s_cross, cross);
  atomicMax(&s_exact, exact);
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double step = a.g.h[0];
  auto xs = [&](int64_t i) { return i == nx - 1 ? a.extent_x : __dmul_rn((double)i, step); };
  double tip, found;
  if (s_cross < 0) {
    found = s_exact >= 0 ? 1.0 : 0.0;
    tip = s_exact >= 0 ? xs(s_exact) : xs(0);
  } else {
    const int64_t i = s_cross;
    const double d0 = __dsub_rn(a.nw[i], a.level), d1 = __dsub_rn(a.nw[i + 1], a.level);
    const double frac = __ddiv_rn(d0, __dsub_rn(d0, d1));
    tip = __dadd_rn(xs(i), __dmul_rn(frac, __dsub_rn(xs(i + 1), xs(i))));
    found = 1.0;
  }
  a.out[D_TIP] = tip;
  a.out[D_FOUND] = found;
}

// map_u_to_c (alloy.py:119-127): composition / (2k) * (1 + k - (1 - k) phi) * (1 + (1 - k) u)
__global__ void k_composition(int64_t n, const double* __restrict__ st, double c2k, double k,
                              double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double omk = 1.0 - k, opk = 1.0 + k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __dmul_rn(__dmul_rn(c2k, __dsub_rn(opk, __dmul_rn(omk, st[i]))),
                       __dadd_rn(1.0, __dmul_rn(omk, st[n + i])));
}

static unsigned diag_grid(int64_t n) {
  int64_t b = (n + UC_DIAG_THREADS * 8 - 1) / (UC_DIAG_THREADS * 8);
  if (b < 1) b = 1;
  if (b > UC_DIAG_GRID_MAX) b = UC_DIAG_GRID_MAX;
  return (unsigned)b;
}

int step_diagnostics(uc_ctx* c, const double* unew, const double* old, const double* prev,
                     const uc_diag_args* in, double* out) {
  if (!c->diag_ws) {
    UC_CUDA_OK(cudaMalloc(&c->diag_ws, sizeof(double) * 6 * UC_DIAG_GRID_MAX + 64));
    UC_CUDA_OK(cudaMemsetAsync(c->diag_ws, 0, sizeof(double) * 6 * UC_DIAG_GRID_MAX + 64, c->stream));
  }
  DiagArgs a{};
  a.g = c->grid;
  a.nw = unew;
  a.od = old;
  a.pv = prev;
  a.ghi = c->ghost[0][1];
  for (int l = 0; l < 8; ++l) a.enw[l] = in->elem_node_weight[l];
  make_jxw(c->grid, a.jxw);
  a.comp_over_2k = in->composition / (2.0 * c->params.kpart);
  a.kpart = c->params.kpart;
  a.level = in->tip_level;
  a.extent_x = in->extent_x;
  a.ws = c->diag_ws;
  a.ticket = (unsigned int*)(c->diag_ws + 6 * UC_DIAG_GRID_MAX);
  a.out = out;
  UC_CUDA_OK(cudaMemsetAsync(out, 0, sizeof(double) * UC_DIAG_N, c->stream));
  const bool balance = (in->what & UC_DIAG_BALANCE) != 0;
  if (balance && (!old || !prev)) return set_error(UC_ERR_ARG, "uc_step_diagnostics: balance needs old and prev");
  k_diag_nodes<<<diag_grid(a.g.nloc), UC_DIAG_THREADS, 0, c->stream>>>(a, balance ? 1 : 0);
  UC_CUDA_OK(cudaGetLastError());
  if (in->what & UC_DIAG_SOLUTE) {
    const Grid& g = a.g;
    const int64_t lay_end = g.hi < g.eslow ? g.hi : g.eslow;
    if (lay_end > g.lo) {
      const int64_t ne = (lay_end - g.lo) * g.ne[0] * (g.dim == 3 ? g.ne[1] : 1);
      if (g.dim == 3)
        k_diag_solute<3><<<diag_grid(ne), UC_DIAG_THREADS, 0, c->stream>>>(a);
      else
        k_diag_solute<2><<<diag_grid(ne), UC_DIAG_THREADS, 0, c->stream>>>(a);
      UC_CUDA_OK(cudaGetLastError());
    }
  }
  if ((in->what & UC_DIAG_TIP) && a.g.lo == 0 && a.g.dim == 2) {
    k_diag_tip<<<1, 1024, 0, c->stream>>>(a);
    UC_CUDA_OK(cudaGetLastError());
  }
  return UC_OK;
}

}  // namespace uc

using namespace uc;

extern "C" int uc_step_diagnostics(uc_ctx* c, const double* unew, const double* old,
                                   const double* prev, const uc_diag_args* args, double* out) {
  if (!c || !unew || !args || !out) return set_error(UC_ERR_ARG, "uc_step_diagnostics: bad argument");
  if ((args->what & UC_DIAG_SOLUTE) && c->grid.hi < c->grid.nslow)
    return set_error(UC_ERR_ARG, "uc_step_diagnostics: slab needs the group entry point (ghost plane)");
  return step_diagnostics(c, unew, old, prev, args, out);
}

extern "C" int uc_map_u_to_c(uc_ctx* c, const double* state, double composition, double* out) {
  if (!c || !state || !out) return set_error(UC_ERR_ARG, "uc_map_u_to_c: bad argument");
  const int64_t n = c->grid.nloc;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)c->num_sms * 16) blocks = (int64_t)c->num_sms * 16;
  if (blocks < 1) blocks = 1;
  k_composition<<<(unsigned)blocks, 256, 0, c->stream>>>(n, state, composition / (2.0 * c->params.kpart),
                                                         c->params.kpart, out);
  UC_CUDA_OK(cudaGetLastError());
  return UC_OK;
}

extern "C" int uc_step_diagnostics_group(uc_ctx* const* ctxs, int n, const double* const* unew,
                                         const double* const* old, const double* const* prev,
                                         const uc_diag_args* args, double* const* out) {
  if (!ctxs || n < 1 || !unew || !args || !out) return set_error(UC_ERR_ARG, "uc_step_diagnostics_group: bad argument");
  Group G(ctxs, ctxs + n);
  if (args->what & UC_DIAG_SOLUTE) {
    const int rc = halo_vectors(G, 0, unew, ctxs[0]->stream);
    if (rc != UC_OK) return rc;
  }
  for (int i = 0; i < n; ++i) {
    const int rc = step_diagnostics(ctxs[i], unew[i], old ? old[i] : nullptr,
                                    prev ? prev[i] : nullptr, args, out[i]);
    if (rc != UC_OK) return rc;
  }
  return UC_OK;
}

// Single-field theta-method mass + diffusion model on the device.
//
// This is the reference's assembly test plug-in `MassDiffKernel`
// (tests/test_assembly.py:22-49):
//   new level:  r0 = u/dt (mass) or 0,    r1 = theta * c * grad u
//   old level:  r0 = -u_old/dt or 0,      r1 = (1 - theta) * c * grad u_old
// integrated with the 3-point Gauss rule and scattered as
// elem_i = r0 @ (psi_i jxw) + sum_d r1_d @ (d_d psi_i jxw) (assembly.py:147-171).
//
// It is not a hot path: one thread per owned node gathers the 2^dim elements
// around it in increasing element order (the order np.bincount sums them),
// so the result is deterministic without atomics.  Single slab only.
#include "uc_internal.h"

namespace uc {
namespace {

struct MdArgs {
  Grid g;
  double jxw[27];
  double inv_dt_s;  // +-mass/dt
  double wc;        // weight * diffusivity
  bool mass;
  const double* u;    // field at the level being assembled (NEW/OLD), or u of Jv
  const double* v;    // Jv direction
  const double* fixed;
  const double* fu;
  double* out;
  unsigned int* flag;
  double eps_num;
  const double* vnorm;
  double* eps_out;
  const uint8_t* emask;  // element subset (assemble_residual(elements=...)); NULL = all
};

// value / gradient weight of local node j = jx + 2jy (+4jz) at qp (qx, qy, qz)
template <int DIM>
__device__ __forceinline__ double psi(int j, const int (&q)[3]) {
  double p = lq(j & 1, q[0]) * lq((j >> 1) & 1, q[1]);
  if (DIM == 3) p = p * lq((j >> 2) & 1, q[2]);
  return p;
}
template <int DIM>
__device__ __forceinline__ double dpsi(const Grid& g, int j, int d, const int (&q)[3]) {
  double p = dsg((j >> d) & 1) * g.ih[d];
#pragma unroll
  for (int b = 0; b < DIM; ++b)
    if (b != d) p = p * lq((j >> b) & 1, q[b]);
  return p;
}

// integrand parts at one qp: r[0] value term, r[1..DIM] flux components
template <int DIM>
__device__ __forceinline__ void qp_terms(const MdArgs& a, const double (&s)[8], const int (&q)[3],
                                         double (&r)[4]) {
  constexpr int NL = 1 << DIM;
  double val = 0.0;
#pragma unroll
  for (int j = 0; j < NL; ++j) val += s[j] * psi<DIM>(j, q);
  r[0] = a.mass ? val * a.inv_dt_s : 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    double gd = 0.0;
#pragma unroll
    for (int j = 0; j < NL; ++j) gd += s[j] * dpsi<DIM>(a.g, j, d, q);
    r[1 + d] = a.wc * gd;
  }
}

template <int DIM>
__device__ __forceinline__ void element_nodes(const MdArgs& a, int64_t ex, int64_t ey, int64_t ez,
                                              double eps, double (&s)[8]) {
  const Grid& g = a.g;
#pragma unroll
  for (int j = 0; j < (1 << DIM); ++j) {
    const int64_t n = (ex + (j & 1)) + (ey + ((j >> 1) & 1)) * g.nn[0] +
                      (DIM == 3 ? (ez + ((j >> 2) & 1)) * g.nn[0] * g.nn[1] : 0);
    s[j] = a.v ? __dadd_rn(a.u[n], __dmul_rn(eps, a.v[n])) : a.u[n];
  }
}

template <int DIM, int MODE>
__global__ void k_massdiff(const __grid_constant__ MdArgs a) {
  const Grid& g = a.g;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double eps = 0.0;
  if (MODE == MODE_JV) {
    const double vn = *a.vnorm;
    if (vn == 0.0) {  // jfnk_matvec returns zeros (newton.py:91-92)
      if (i < g.nloc) a.out[i] = 0.0;
      if (a.eps_out && i == 0) *a.eps_out = 0.0;
      return;
    }
    eps = a.eps_num / vn;
    if (a.eps_out && i == 0) *a.eps_out = eps;
  }
  if (i >= g.nloc) return;
  const int64_t ix = i % g.nn[0];
  const int64_t iy = DIM == 3 ? (i / g.nn[0]) % g.nn[1] : i / g.nn[0];
  const int64_t iz = DIM == 3 ? i / (g.nn[0] * g.nn[1]) : 0;
  constexpr int NQ1 = 3, NQ = DIM == 3 ? 27 : 9;
  double live = 0.0;
  for (int bz = 0; bz < (DIM == 3 ? 2 : 1); ++bz) {
    const int64_t ez = iz - 1 + bz;
    if (DIM == 3 && (ez < 0 || ez >= g.ne[2])) continue;
    for (int by = 0; by < 2; ++by) {
      const int64_t ey = iy - 1 + by;
      if (ey < 0 || ey >= g.ne[1]) continue;
      for (int bx = 0; bx < 2; ++bx) {
        const int64_t ex = ix - 1 + bx;
        if (ex < 0 || ex >= g.ne[0]) continue;
        if (a.emask && !a.emask[ex + ey * g.ne[0] + (DIM == 3 ? ez * g.ne[0] * g.ne[1] : 0)]) continue;
        double s[8];
        element_nodes<DIM>(a, ex, ey, DIM == 3 ? ez : 0, eps, s);
        const int me = (1 - bx) + 2 * (1 - by) + (DIM == 3 ? 4 * (1 - bz) : 0);
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        for (int qq = 0; qq < NQ; ++qq) {
          const int q[3] = {qq % NQ1, (qq / NQ1) % NQ1, qq / (NQ1 * NQ1)};
          double r[4];
          qp_terms<DIM>(a, s, q, r);
          t[0] += r[0] * (psi<DIM>(me, q) * a.jxw[qq]);
#pragma unroll
          for (int d = 0; d < DIM; ++d) t[1 + d] += r[1 + d] * (dpsi<DIM>(g, me, d, q) * a.jxw[qq]);
        }
        double e = t[0];
#pragma unroll
        for (int d = 0; d < DIM; ++d) e += t[1 + d];
        live += e;
      }
    }
  }
  if (!isfinite(live)) *(volatile unsigned int*)a.flag = 1u;
  if (MODE == MODE_OLD)
    a.out[i] = live;
  else if (MODE == MODE_NEW)
    a.out[i] = a.fixed ? live + a.fixed[i] : live;
  else
    a.out[i] = __dsub_rn(live + a.fixed[i], a.fu[i]) / eps;
}

// smallest (part, element, qp) key with a non-finite integrand
template <int DIM>
__global__ void k_massdiff_locate(const __grid_constant__ MdArgs a, unsigned long long* key) {
  const Grid& g = a.g;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ne = g.ne[0] * g.ne[1] * (DIM == 3 ? g.ne[2] : 1);
  if (e >= ne || (a.emask && !a.emask[e])) return;
  const int64_t ex = e % g.ne[0];
  const int64_t ey = DIM == 3 ? (e / g.ne[0]) % g.ne[1] : e / g.ne[0];
  const int64_t ez = DIM == 3 ? e / (g.ne[0] * g.ne[1]) : 0;
  double s[8];
  element_nodes<DIM>(a, ex, ey, ez, 0.0, s);
  unsigned long long best = ~0ull;
  constexpr int NQ = DIM == 3 ? 27 : 9;
  for (int qq = 0; qq < NQ; ++qq) {
    const int q[3] = {qq % 3, (qq / 3) % 3, qq / 9};
    double r[4];
    qp_terms<DIM>(a, s, q, r);
    for (int w = 0; w <= DIM; ++w)
      if (!isfinite(r[w])) {
        const unsigned long long k =
            ((unsigned long long)w << 44) | ((unsigned long long)e << 5) | (unsigned long long)qq;
        best = k < best ? k : best;
      }
  }
  if (best != ~0ull) atomicMin(key, best);
}

MdArgs make_md(uc_ctx* c, const uc_scheme* sc, int mode) {
  MdArgs a{};
  a.g = c->grid;
  make_jxw(c->grid, a.jxw);
  const bool newlvl = mode != MODE_OLD;
  const double weight = newlvl ? sc->theta : 1.0 - sc->theta;
  a.inv_dt_s = (newlvl ? 1.0 : -1.0) / sc->dt;
  a.wc = weight * c->params.dcoef;
  a.mass = c->params.mass_coef != 0.0;
  a.flag = c->flags;
  return a;
}

}  // namespace

int launch_massdiff(uc_ctx* c, const uc_scheme* sc, int mode, const double* u, const double* old,
                    const double* v, const double* fu, const double* fixed, double* out,
                    double eps_num, const double* vnorm_dev, double* eps_out) {
  MdArgs a = make_md(c, sc, mode);
  a.u = mode == MODE_OLD ? old : u;
  a.v = mode == MODE_JV ? v : nullptr;
  a.fu = fu;
  a.fixed = fixed;
  a.out = out;
  a.eps_num = eps_num;
  a.vnorm = vnorm_dev;
  a.eps_out = eps_out;
  const unsigned blocks = (unsigned)((c->grid.nloc + 255) / 256);
  const bool d2 = c->grid.dim == 2;
  if (mode == MODE_OLD)
    d2 ? k_massdiff<2, MODE_OLD><<<blocks, 256, 0, c->stream>>>(a)
       : k_massdiff<3, MODE_OLD><<<blocks, 256, 0, c->stream>>>(a);
  else if (mode == MODE_NEW)
    d2 ? k_massdiff<2, MODE_NEW><<<blocks, 256, 0, c->stream>>>(a)
       : k_massdiff<3, MODE_NEW><<<blocks, 256, 0, c->stream>>>(a);
  else
    d2 ? k_massdiff<2, MODE_JV><<<blocks, 256, 0, c->stream>>>(a)
       : k_massdiff<3, MODE_JV><<<blocks, 256, 0, c->stream>>>(a);
  UC_CUDA_OK(cudaGetLastError());
  return UC_OK;
}

int launch_massdiff_subset(uc_ctx* c, const uc_scheme* sc, int mode, const double* u,
                           const double* old, const double* fixed, const uint8_t* emask, double* out) {
  MdArgs a = make_md(c, sc, mode);
  a.u = mode == MODE_OLD ? old : u;
  a.fixed = fixed;
  a.out = out;
  a.emask = emask;
  const unsigned blocks = (unsigned)((c->grid.nloc + 255) / 256);
  const bool d2 = c->grid.dim == 2;
  if (mode == MODE_OLD)
    d2 ? k_massdiff<2, MODE_OLD><<<blocks, 256, 0, c->stream>>>(a)
       : k_massdiff<3, MODE_OLD><<<blocks, 256, 0, c->stream>>>(a);
  else
    d2 ? k_massdiff<2, MODE_NEW><<<blocks, 256, 0, c->stream>>>(a)
       : k_massdiff<3, MODE_NEW><<<blocks, 256, 0, c->stream>>>(a);
  UC_CUDA_OK(cudaGetLastError());
  return UC_OK;
}

int locate_massdiff(uc_ctx* c, const uc_scheme* sc, int mode, const double* u, const double* old,
                    const uint8_t* emask, unsigned long long* key_dev) {
  MdArgs a = make_md(c, sc, mode);
  a.emask = emask;
  a.u = mode == MODE_OLD ? old : u;
  const Grid& g = c->grid;
  const int64_t ne = g.ne[0] * g.ne[1] * (g.dim == 3 ? g.ne[2] : 1);
  const unsigned blocks = (unsigned)((ne + 127) / 128);
  if (g.dim == 2)
    k_massdiff_locate<2><<<blocks, 128, 0, c->stream>>>(a, key_dev);
  else
    k_massdiff_locate<3><<<blocks, 128, 0, c->stream>>>(a, key_dev);
  UC_CUDA_OK(cudaGetLastError());
  return UC_OK;
}

}  // namespace uc

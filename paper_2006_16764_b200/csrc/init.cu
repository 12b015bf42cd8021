// On-device initial conditions: the host versions need
// the full coordinate array (3.2 GB at 512^3).  Each context fills its owned
// node planes.
//
//   seed         free_growth.py:249-265: phi = [|x| <= r g(x)], T = T_far,
//                g = fourfold(x) with the default blend scale (anisotropy.py:23-68)
//   directional  alloy.py:317-357: corrugated planar interface from a
//                splitmix64 counter per transverse row, tanh or sharp profile,
//                u = -1
#include "uc_internal.h"

namespace uc {

struct InitArgs {
  Grid g;
  double extent[3];
  double step[3];  // linspace step = extent / counts
  int kind;        // 0 seed, 1 directional
  double eps, radius, t_far;            // seed
  double x0, amplitude;                 // directional
  unsigned long long seed;
  int smooth;
  double* out;
};

// node coordinate along axis a exactly as numpy.linspace builds it
__device__ __forceinline__ double lin_coord(const InitArgs& a, int ax, int64_t i) {
  return i == a.g.nn[ax] - 1 ? a.extent[ax] : __dmul_rn((double)i, a.step[ax]);
}

__device__ __forceinline__ double splitmix_unit(unsigned long long seed, unsigned long long idx) {
  unsigned long long z = (seed + idx + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return (double)(z >> 11) / 9007199254740992.0;  // / 2^53
}

__global__ void k_initial(const InitArgs a) {
  const Grid& g = a.g;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.nloc; q += stride) {
    const int64_t gid = g.lo * g.plane + q;  // global node id
    const int64_t i0 = gid % g.nn[0];
    const int64_t r = gid / g.nn[0];
    double x[3];
    x[0] = lin_coord(a, 0, i0);
    if (g.dim == 3) {
      x[1] = lin_coord(a, 1, r % g.nn[1]);
      x[2] = lin_coord(a, 2, r / g.nn[1]);
    } else {
      x[1] = lin_coord(a, 1, r);
    }
    double phi, sec;
    if (a.kind == 0) {
      // fourfold(x, eps) with reg_grad = 1e-3 and |x| (numpy operation order)
      double p2[3], s2 = 0.0, quart = 0.0;
      for (int d = 0; d < g.dim; ++d) {
        p2[d] = __dmul_rn(x[d], x[d]);
        s2 = d == 0 ? p2[0] : __dadd_rn(s2, p2[d]);
        const double p4 = __dmul_rn(p2[d], p2[d]);
        quart = d == 0 ? p4 : __dadd_rn(quart, p4);
      }
      const double reg = 1e-12;  // GRAD_REG**4
      const double avg = g.dim == 3 ? 1.0 / 3.0 : 0.5;
      const double denom = __dadd_rn(__dmul_rn(s2, s2), reg);
      const double ratio = __ddiv_rn(__dadd_rn(quart, __dmul_rn(avg, reg)), denom);
      const double gg = __dadd_rn(__dsub_rn(1.0, __dmul_rn(3.0, a.eps)), __dmul_rn(__dmul_rn(4.0, a.eps), ratio));
      const double dist = __dsqrt_rn(s2);
      phi = dist <= __dmul_rn(a.radius, gg) ? 1.0 : 0.0;
      sec = a.t_far;
    } else {
      const double xi = __dsub_rn(__dmul_rn(2.0, splitmix_unit(a.seed, (unsigned long long)r)), 1.0);
      const double thr = __dadd_rn(a.x0, __dmul_rn(a.amplitude, xi));
      if (a.smooth)
        phi = tanh(__ddiv_rn(__dsub_rn(thr, x[0]), sqrt(2.0)));
      else
        phi = x[0] <= thr ? 1.0 : -1.0;
      sec = -1.0;
    }
    a.out[q] = phi;
    a.out[g.nloc + q] = sec;
  }
}

}  // namespace uc

using namespace uc;

// params: seed {eps, radius, t_far}; directional {x0, amplitude, seed, smooth}
extern "C" int uc_initial_state(uc_ctx* c, int kind, const double* extents, const double* params,
                                double* out) {
  if (!c || !extents || !params || !out || kind < 0 || kind > 1)
    return set_error(UC_ERR_ARG, "uc_initial_state: bad argument");
  InitArgs a{};
  a.g = c->grid;
  for (int d = 0; d < 3; ++d) {
    a.extent[d] = d < a.g.dim ? extents[d] : 1.0;
    a.step[d] = d < a.g.dim ? extents[d] / (double)a.g.ne[d] : 1.0;
  }
  a.kind = kind;
  if (kind == 0) {
    a.eps = params[0];
    a.radius = params[1];
    a.t_far = params[2];
  } else {
    a.x0 = params[0];
    a.amplitude = params[1];
    a.seed = (unsigned long long)params[2];
    a.smooth = params[3] != 0.0;
  }
  a.out = out;
  int64_t blocks = (a.g.nloc + 255) / 256;
  if (blocks > (int64_t)c->num_sms * 32) blocks = (int64_t)c->num_sms * 32;
  k_initial<<<(unsigned)blocks, 256, 0, c->stream>>>(a);
  UC_CUDA_OK(cudaGetLastError());
  return UC_OK;
}

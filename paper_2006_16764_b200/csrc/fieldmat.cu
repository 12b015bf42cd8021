// Quadrature-point interpolation and the field mass+stiffness matrix as
// device operations of the drop-in surface:
//
//   uc_quad_state      frozen_quad_state (undercool/assembly.py:193-211 via
//                      _interp :111-116 and StructuredMesh.gauss_coords
//                      mesh.py:119-128): per element and quadrature point the
//                      field values, physical gradients and coordinates.
//   uc_field_matrix    assemble_field_matrix (assembly.py:271-303):
//                      (cmass psi_j, psi_i) + (cdiff grad psi_j, grad psi_i)
//                      with per-quadrature-point (or scalar) coefficients,
//                      written straight into CSR (rows sorted, structural
//                      entries of every element coupling, duplicates summed in
//                      element-id order as COO->CSR does).
//
// Any tensor Gauss rule: the basis tables (values, physical gradients, jxw of
// mesh.py:151-176 for the rule, nq points) come in from the caller.  Whole
// (unsplit) meshes only.
#include "uc_internal.h"

namespace uc {

struct BasisDev {
  const double* V;   // [nq][nloc]
  const double* G;   // [nq][nloc][dim]
  const double* W;   // [nq] jxw
  const double* P;   // [nq][dim] reference points in [-1, 1]
  int nq, nloc, dim;
};

// one thread per (element, quadrature point); element-major output
__global__ void k_quad_state(const Grid g, const BasisDev b, const double* __restrict__ state, int nf,
                             double* __restrict__ coords, double* __restrict__ vals, double* __restrict__ grads) {
  const int64_t ne = g.ne[0] * g.ne[1] * g.ne[2];
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ne * b.nq) return;
  const int64_t e = t / b.nq;
  const int q = (int)(t - e * b.nq);
  const int64_t e0 = e % g.ne[0], r = e / g.ne[0];
  const int64_t e1 = g.dim == 3 ? r % g.ne[1] : r, e2 = g.dim == 3 ? r / g.ne[1] : 0;
  const int64_t nx = g.nn[0], nxy = g.nn[0] * g.nn[1];
  const int64_t n0 = e0 + nx * e1 + nxy * e2;  // lowest-corner node (conn[:, 0])
  const int64_t N = g.plane * g.nslow;
  for (int f = 0; f < nf; ++f) {
    const double* u = state + f * N;
    double v = 0.0, gd[3] = {0.0, 0.0, 0.0};
    for (int loc = 0; loc < b.nloc; ++loc) {
      const int64_t node = n0 + (loc & 1) + nx * ((loc >> 1) & 1) + nxy * ((loc >> 2) & 1);
      const double un = u[node];
      v = __dadd_rn(v, __dmul_rn(un, b.V[q * b.nloc + loc]));
      for (int d = 0; d < g.dim; ++d) gd[d] = __dadd_rn(gd[d], __dmul_rn(un, b.G[(q * b.nloc + loc) * g.dim + d]));
    }
    vals[(int64_t)f * ne * b.nq + t] = v;
    for (int d = 0; d < g.dim; ++d) grads[((int64_t)f * g.dim + d) * ne * b.nq + t] = gd[d];
  }
  if (coords) {
    const int64_t ei[3] = {e0, e1, e2};
    for (int d = 0; d < g.dim; ++d) {
      // origin = node coordinate (i * h, == linspace bitwise), local = (p + 1) / 2 * h
      const double org = __dmul_rn((double)ei[d], g.h[d]);
      const double loc = __dmul_rn(__dmul_rn(__dadd_rn(b.P[q * g.dim + d], 1.0), 0.5), g.h[d]);
      coords[(t * g.dim) + d] = __dadd_rn(org, loc);
    }
  }
}

// number of stencil neighbours of node i along an axis of n nodes
__device__ __forceinline__ int64_t ncount(int64_t i, int64_t n) { return 1 + (i > 0) + (i < n - 1); }
// sum of ncount over nodes 0..i-1
__device__ __forceinline__ int64_t nprefix(int64_t i, int64_t n) {
  return i + (i > 0 ? i - 1 : 0) + (i < n - 1 ? i : n - 1);
}

// one thread per row: the row's structural entries in ascending column order,
// each the sum over the elements sharing (row, column) in element-id order
__global__ void k_field_csr(const Grid g, const BasisDev b, const double* __restrict__ cm, int64_t cms,
                            const double* __restrict__ cd, int64_t cds, int64_t* __restrict__ indptr,
                            int32_t* __restrict__ indices, double* __restrict__ data) {
  const int64_t N = g.plane * g.nslow;
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row > N) return;
  const int dim = g.dim;
  const int64_t n[3] = {g.nn[0], g.nn[1], dim == 3 ? g.nn[2] : 1};
  const int64_t T0 = nprefix(n[0], n[0]), T1 = nprefix(n[1], n[1]);
  if (row == N) {
    indptr[N] = T0 * T1 * (dim == 3 ? nprefix(n[2], n[2]) : 1);
    return;
  }
  const int64_t i0 = row % n[0], rr = row / n[0];
  const int64_t i1 = dim == 3 ? rr % n[1] : rr, i2 = dim == 3 ? rr / n[1] : 0;
  const int64_t c0 = ncount(i0, n[0]), c1 = ncount(i1, n[1]);
  int64_t start = nprefix(i0, n[0]) * c1 + T0 * nprefix(i1, n[1]);
  if (dim == 3) start = start * ncount(i2, n[2]) + T0 * T1 * nprefix(i2, n[2]);
  indptr[row] = start;
  const int nz = dim == 3 ? 3 : 1;
  int64_t out = start;
  for (int dz = (dim == 3 ? -1 : 0); dz <= (dim == 3 ? 1 : 0); ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int64_t j0 = i0 + dx, j1 = i1 + dy, j2 = i2 + dz;
        if (j0 < 0 || j0 >= n[0] || j1 < 0 || j1 >= n[1] || j2 < 0 || j2 >= n[2]) continue;
        double acc = 0.0;
        bool first = true;
        // elements containing both nodes, in element-id order (z, y, x slowest first)
        for (int az = 0; az < (dim == 3 ? 2 : 1); ++az)
          for (int ay = 0; ay < 2; ++ay)
            for (int ax = 0; ax < 2; ++ax) {
              const int64_t E0 = i0 - 1 + ax, E1 = i1 - 1 + ay, E2 = dim == 3 ? i2 - 1 + az : 0;
              if (E0 < 0 || E0 >= g.ne[0] || E1 < 0 || E1 >= g.ne[1] || E2 < 0 || E2 >= g.ne[2]) continue;
              const int li0 = (int)(i0 - E0), li1 = (int)(i1 - E1), li2 = (int)(i2 - E2);
              const int lj0 = (int)(j0 - E0), lj1 = (int)(j1 - E1), lj2 = (int)(j2 - E2);
              if (lj0 < 0 || lj0 > 1 || lj1 < 0 || lj1 > 1 || lj2 < 0 || lj2 > 1) continue;
              const int li = li0 + 2 * li1 + 4 * li2, lj = lj0 + 2 * lj1 + 4 * lj2;
              const int64_t e = E0 + g.ne[0] * (E1 + g.ne[1] * E2);
              double m = 0.0, k = 0.0;
              for (int q = 0; q < b.nq; ++q) {
                const double w = b.W[q];
                const double cmq = __dmul_rn(cm[cms ? e * cms + q : 0], w);
                const double cdq = __dmul_rn(cd[cds ? e * cds + q : 0], w);
                m = __dadd_rn(m, __dmul_rn(__dmul_rn(cmq, b.V[q * b.nloc + li]), b.V[q * b.nloc + lj]));
                double gg = 0.0;
                for (int d = 0; d < dim; ++d)
                  gg = __dadd_rn(gg, __dmul_rn(b.G[(q * b.nloc + li) * dim + d], b.G[(q * b.nloc + lj) * dim + d]));
                k = __dadd_rn(k, __dmul_rn(cdq, gg));
              }
              const double ev = __dadd_rn(m, k);
              acc = first ? ev : __dadd_rn(acc, ev);
              first = false;
            }
        indices[out] = (int32_t)(j0 + n[0] * (j1 + n[1] * j2));
        data[out] = acc;
        ++out;
      }
  (void)nz;
  (void)c0;
}

}  // namespace uc

using namespace uc;

static BasisDev basis_dev(const uc_ctx* c, const double* tables, int nq) {
  BasisDev b;
  b.dim = c->grid.dim;
  b.nq = nq;
  b.nloc = 1 << b.dim;
  b.V = tables;
  b.G = tables + nq * b.nloc;
  b.W = b.G + nq * b.nloc * b.dim;
  b.P = b.W + nq;
  return b;
}

extern "C" {

int uc_quad_state(uc_ctx* c, const double* state, int nfields, const double* tables, int nq, double* coords,
                  double* vals, double* grads) {
  if (!c || !state || !tables || !vals || !grads || nq < 1 || nfields < 1)
    return set_error(UC_ERR_ARG, "uc_quad_state: bad argument");
  if (c->grid.lo != 0 || c->grid.hi != c->grid.nslow)
    return set_error(UC_ERR_UNSUPPORTED, "uc_quad_state: whole meshes only");
  const Grid& g = c->grid;
  const int64_t work = g.ne[0] * g.ne[1] * g.ne[2] * nq;
  if (work == 0) return UC_OK;
  k_quad_state<<<(unsigned)((work + 255) / 256), 256, 0, c->stream>>>(g, basis_dev(c, tables, nq), state, nfields,
                                                                     coords, vals, grads);
  UC_CUDA_OK(cudaGetLastError());
  return UC_OK;
}

int64_t uc_field_matrix_nnz(uc_ctx* c) {
  if (!c) return -1;
  const Grid& g = c->grid;
  auto T = [](int64_t n) { return n + (n > 1 ? n - 1 : 0) + (n > 1 ? n - 1 : 0); };
  return T(g.nn[0]) * T(g.nn[1]) * (g.dim == 3 ? T(g.nn[2]) : 1);
}

int uc_field_matrix(uc_ctx* c, const double* cmass, int64_t cmass_stride, const double* cdiff, int64_t cdiff_stride,
                    const double* tables, int nq, int64_t* indptr, int32_t* indices, double* data) {
  if (!c || !cmass || !cdiff || !tables || !indptr || !indices || !data || nq < 1 || cmass_stride < 0 ||
      cdiff_stride < 0)
    return set_error(UC_ERR_ARG, "uc_field_matrix: bad argument");
  if (c->grid.lo != 0 || c->grid.hi != c->grid.nslow)
    return set_error(UC_ERR_UNSUPPORTED, "uc_field_matrix: whole meshes only");
  const Grid& g = c->grid;
  const int64_t N = g.plane * g.nslow;
  if (N >= ((int64_t)1 << 31)) return set_error(UC_ERR_UNSUPPORTED, "uc_field_matrix: more than 2^31 rows");
  k_field_csr<<<(unsigned)((N + 1 + 255) / 256), 256, 0, c->stream>>>(g, basis_dev(c, tables, nq), cmass, cmass_stride,
                                                                      cdiff, cdiff_stride, indptr, indices, data);
  UC_CUDA_OK(cudaGetLastError());
  return UC_OK;
}

}  // extern "C"

/*
 * uc_b200.h — C ABI of the B200-native hot path of the Tusas/undercool JFNK
 * phase-field solver (arXiv:2006.16764).
 *
 * All vector arguments are DEVICE pointers to fp64 arrays in the reference's
 * block-by-field layout (all nodes of field 0, then all nodes of field 1;
 * nodes lexicographic with x fastest — undercool/assembly.py:48-54,
 * undercool/mesh.py:209-228).  Every entry point is asynchronous on the
 * context's CUDA stream unless it says it synchronises.  Return codes:
 *
 *   UC_OK (0)            success
 *   UC_ERR_NONFINITE (1) a non-finite value was detected (see uc_status)
 *   UC_ERR_ARG (2)       bad argument (message in uc_last_error())
 *   UC_ERR_CUDA (3)      CUDA / NCCL failure
 *   UC_ERR_UNSUPPORTED (4)
 *
 * The reference is pure Python (numpy/scipy/numba); it has no FFI of its own.
 * Each entry point below names the reference function it replaces; the
 * ctypes binding a maintainer of the reference would add is in
 * INTEGRATION.md.  No torch types appear in this interface.
 */
#ifndef UC_B200_H
#define UC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UC_OK 0
#define UC_ERR_NONFINITE 1
#define UC_ERR_ARG 2
#define UC_ERR_CUDA 3
#define UC_ERR_UNSUPPORTED 4

#define UC_MODEL_FREE_GROWTH 1
#define UC_MODEL_ALLOY 2
#define UC_MODEL_MASS_DIFF 3  /* single-field mass + diffusion test model (tests/test_assembly.py:22-49) */

#define UC_PART_NEW 0
#define UC_PART_OLD 1

#define UC_PC_IDENTITY 0
#define UC_PC_JACOBI 1
#define UC_PC_SGS 2
#define UC_PC_VCYCLE 3

typedef struct uc_ctx uc_ctx;

/* Structured Q1 mesh (undercool/mesh.py:179-256 build_mesh).  spacing[a] must
 * equal extents[a]/counts[a] as the reference computes it.  A rank owns node
 * planes [slab_lo, slab_hi) along the slowest axis (y in 2D, z in 3D); a
 * single GPU owns [0, counts[dim-1]+1). */
typedef struct uc_mesh_desc {
  int32_t dim;
  int32_t order;
  int64_t counts[3];
  double spacing[3];
  int64_t slab_lo;
  int64_t slab_hi;
} uc_mesh_desc;

/* Physics constants, derived on the host exactly as the reference's kernel
 * wrappers derive them (free_growth.py:163-206, alloy.py:225-269). */
typedef struct uc_model_params {
  int32_t model;          /* UC_MODEL_* */
  int32_t normalized;     /* alloy: antitrapping_normalized */
  double eps;             /* anisotropy_strength */
  double reg;             /* aniso_reg_grad**4 */
  double aniso_reg_grad;  /* blend scale used by fourfold() in the preconditioner */
  /* free growth */
  double bg;              /* kinetic_coeff * mobility */
  double beta;            /* kinetic_coeff */
  double alpha;           /* thermal_diffusivity */
  double latent;          /* latent_ratio */
  double hcell;           /* mesh_scale */
  double tmelt;           /* melt_temperature */
  /* alloy */
  double at_reg2;         /* antitrap_reg_grad**2 */
  double kpart;           /* partition */
  double coupling;
  double dcoef;           /* diffusivity */
  double g4_coef;         /* frame_coefficient */
  double pull_velocity;
  /* mass-diffusion (dcoef = diffusivity) */
  double mass_coef;       /* 1: (du/dt, psi) term present, 0: diffusion only */
} uc_model_params;

/* ThetaScheme (undercool/stepping.py:12-37). */
typedef struct uc_scheme {
  double theta;
  double dt;
  int64_t step;
} uc_scheme;

/* PrecondConfig (undercool/precond.py:54-71). */
#define UC_ORDER_MULTICOLOR 0
#define UC_ORDER_LEXICOGRAPHIC 1
#define UC_ORDER_LEXICOGRAPHIC_WAVEFRONT 2  /* same sweep, grid-barrier wavefront kernel (validation) */
#define UC_ORDER_LEXICOGRAPHIC_ROWS 3       /* same sweep, 3D: every row streams its own stencil (validation) */
typedef struct uc_precond_cfg {
  int32_t kind;           /* UC_PC_* */
  int32_t sweeps;
  int32_t cycles;
  int32_t levels;
  int32_t coarse_sweeps;
  int32_t ordering;       /* UC_ORDER_*: lexicographic = exact sequential GS as a wavefront */
} uc_precond_cfg;

/* Sticky device-side status, read with uc_status (synchronises). */
typedef struct uc_status_t {
  int32_t residual_nonfinite;   /* a residual/Jv output entry was non-finite */
  int32_t precond_nonfinite;    /* a preconditioner application was non-finite */
  int32_t precond_bad_diag;     /* build: non-positive (fine) / zero (coarse) diagonal */
  int32_t pad;
} uc_status_t;

int uc_abi_version(void);
const char* uc_last_error(void);

/* Create / destroy a context bound to the current device.  stream may be 0. */
int uc_ctx_create(const uc_mesh_desc* mesh, const uc_model_params* params,
                  void* cuda_stream, uc_ctx** out);
int uc_ctx_destroy(uc_ctx* ctx);
int uc_set_stream(uc_ctx* ctx, void* cuda_stream);
int64_t uc_n_local(const uc_ctx* ctx);  /* owned nodes per field on this rank */

/* Ghost node planes for slab-decomposed runs: device storage for one plane of
 * both fields below (side 0) and above (side 1) the owned slab, per input
 * slot (0 = u/new, 1 = old, 2 = prev, 3 = v).  The host fills them (NCCL
 * send/recv) before a residual/Jv call.  NULL on a single GPU. */
double* uc_ghost_ptr(uc_ctx* ctx, int slot, int side);

/* assemble_residual(part="new"|"old") (assembly.py:214-230) restricted to the
 * owned nodes, with the lagged rate (stepping.py:40-50) built on the fly.
 *   part = UC_PART_OLD: out = old-level assembly (TimestepResidual.fixed_part,
 *          assembly.py:256-258); `unew` is ignored.
 *   part = UC_PART_NEW: out = new-level assembly + fixed (TimestepResidual.
 *          __call__, assembly.py:261-268).
 * A non-finite assembled entry sets residual_nonfinite. */
int uc_residual(uc_ctx* ctx, const uc_scheme* sc, int part, const double* unew,
                const double* old, const double* prev, const double* fixed,
                double* out);

/* Locate the first non-finite Gauss-point integrand like _check_finite
 * (assembly.py:174-190).  Synchronises.  Writes field, part (0 value,
 * 1+d flux[d]), element id, quadrature point and first node; returns 0 if
 * every integrand is finite (fields set to -1). */
/* assemble_residual(..., elements=subset) (assembly.py:214-230 with `elements`):
 * the same parts, summed over the elements whose byte in element_mask
 * (n_elements, element-id order) is non-zero.  part = UC_PART_OLD: out = old
 * level; UC_PART_NEW: out = new level + fixed (fixed may be NULL for the new
 * level alone).  Single slab only; not a hot path (node-centric gather, each
 * element re-evaluated by its corner nodes). */
int uc_residual_subset(uc_ctx* ctx, const uc_scheme* sc, int part, const double* unew,
                       const double* old, const double* prev, const double* fixed,
                       const uint8_t* element_mask, double* out);

/* uc_locate_nonfinite restricted to the elements of element_mask. */
int uc_locate_nonfinite_subset(uc_ctx* ctx, const uc_scheme* sc, int part, const double* unew,
                               const double* old, const double* prev, const uint8_t* element_mask,
                               int64_t* field, int64_t* which, int64_t* element, int64_t* qp,
                               int64_t* first_node);
int uc_locate_nonfinite(uc_ctx* ctx, const uc_scheme* sc, int part,
                        const double* unew, const double* old, const double* prev,
                        int64_t* field, int64_t* which, int64_t* element,
                        int64_t* qp, int64_t* first_node);

/* _FdOperator.__call__ / jfnk_matvec (newton.py:84-113):
 *   jv = (F(u + eps v) - fu) / eps,  eps = sqrt(DBL_EPSILON)*sqrt(1+unorm)/|v|,
 * with u + eps v formed on the fly inside the residual tile.  |v| is reduced
 * on the device; jv = 0 if |v| == 0.  eps_out (device, may be NULL) receives eps
 * (0 when |v| == 0). */
int uc_jv(uc_ctx* ctx, const uc_scheme* sc, const double* u, const double* fu,
          const double* v, double unorm, const double* old, const double* prev,
          const double* fixed, double* jv, double* eps_out);

/* Deterministic fixed-order reductions over n entries (np.dot / np.linalg.norm
 * as used by newton.py and krylov.py).  Results go to device scalars. */
int uc_dot(uc_ctx* ctx, int64_t n, const double* a, const double* b, double* out_dev);
int uc_norm(uc_ctx* ctx, int64_t n, const double* a, double* out_dev);
/* Host-returning variants (synchronise). */
int uc_dot_host(uc_ctx* ctx, int64_t n, const double* a, const double* b, double* out);
int uc_norm_host(uc_ctx* ctx, int64_t n, const double* a, double* out);

/* arnoldi_step (krylov.py:48-70): MGS of w against basis[0..k] plus one full
 * re-orthogonalisation pass, h[k+1] = |w|, and basis[k+1] = w / h[k+1] unless
 * h[k+1] < 1e-14*scale (breakdown).  basis is an array of k+2 device pointers
 * (basis[k+1] is the output slot).  Synchronises; h_host gets k+2 values,
 * *broke the breakdown flag. */
int uc_arnoldi(uc_ctx* ctx, int64_t n, const double* const* basis, int k,
               double* w, double scale, double* h_host, int* broke);

/* arnoldi_step with classical Gram-Schmidt applied twice (CGS2): the same
 * projections as uc_arnoldi's MGS + re-orthogonalisation (krylov.py:48-70)
 * computed pass-wise, so a distributed step needs two (k+1)-value global sums
 * and one norm instead of 2(k+1) scalar sums.  Opt-in
 * (GmresConfig.orthogonalization = "cgs2"); k + 1 <= 256. */
int uc_arnoldi_cgs2(uc_ctx* ctx, int64_t n, const double* const* basis, int k, double* w,
                    double scale, double* h_host, int* broke);
int uc_arnoldi_cgs2_group(uc_ctx* const* ctxs, int nslabs, const double* const* basis, int k,
                          double* const* w, double scale, double* h_host, int* broke);

/* out = sum_j y[j] * basis[j], j = 0..k-1 (krylov.py:180-182 basis[:k].T @ y). */
int uc_combine(uc_ctx* ctx, int64_t n, const double* const* basis, int k,
               const double* y_host, double* out);

/* Elementwise helpers used by the solver control flow (newton.py:164-165,
 * krylov.py:124-131,183,191): out = a + s*b  (two roundings, numpy order). */
int uc_axpy(uc_ctx* ctx, int64_t n, const double* a, double s, const double* b,
            double* out);
/* out = a - b */
int uc_sub(uc_ctx* ctx, int64_t n, const double* a, const double* b, double* out);
/* out = a / s */
int uc_scale_div(uc_ctx* ctx, int64_t n, const double* a, double s, double* out);
/* out = s * a */
int uc_scale(uc_ctx* ctx, int64_t n, double s, const double* a, double* out);
/* frozen_quad_state (undercool/assembly.py:193-211, _interp :111-116,
 * gauss_coords mesh.py:119-128) of a whole mesh: for every element e and
 * quadrature point q of the rule, vals[f][e][q], grads[f][d][e][q] and
 * coords[e][q][d] (coords may be NULL).  tables = [values nq x nloc |
 * physical gradients nq x nloc x dim | jxw nq | reference points nq x dim]
 * (mesh.py:151-176) on the device. */
int uc_quad_state(uc_ctx* ctx, const double* state, int nfields, const double* tables, int nq,
                  double* coords, double* vals, double* grads);
/* assemble_field_matrix (assembly.py:271-303): (cmass psi_j, psi_i) +
 * (cdiff grad psi_j, grad psi_i) in CSR (n_nodes + 1 row pointers, int32
 * column indices sorted per row, one entry per element coupling, duplicates
 * summed).  cmass/cdiff: per (element, quadrature point) with stride nq, or
 * one scalar with stride 0.  uc_field_matrix_nnz gives the entry count. */
int64_t uc_field_matrix_nnz(uc_ctx* ctx);
int uc_field_matrix(uc_ctx* ctx, const double* cmass, int64_t cmass_stride, const double* cdiff,
                    int64_t cdiff_stride, const double* tables, int nq, int64_t* indptr, int32_t* indices,
                    double* data);

/* Host-visible vector tests of the Newton control flow (newton.py:144,175-176
 * np.all(np.isfinite(x)), np.any(x)): *nonfinite = 1 if some entry is NaN/Inf,
 * *nonzero = 1 if some entry is non-zero.  Synchronises the context stream. */
int uc_vec_check(uc_ctx* ctx, int64_t n, const double* a, int32_t* nonfinite, int32_t* nonzero);

/* build_precond (precond.py:269-299): frozen Gauss-point state -> block
 * coefficients (free_growth.py:223-231 / alloy.py:286-300) -> fixed 9/27-point
 * stencils (assembly.py:271-303) -> Galerkin hierarchy (precond.py:191-206).
 * Synchronises; returns UC_ERR_ARG with precond_bad_diag set on a
 * non-positive diagonal. */
int uc_precond_build(uc_ctx* ctx, const uc_scheme* sc, const double* state,
                     const uc_precond_cfg* cfg);
/* BlockPrecond.apply (precond.py:248-264), both field blocks per launch. */
int uc_precond_apply(uc_ctx* ctx, const double* v, double* out);
/* Copy the stencil of level/block to host: rows x 3^dim values in natural
 * row order, offsets (dx,dy[,dz]) lexicographic with dx fastest. */
int uc_precond_stencil(uc_ctx* ctx, int level, int block, double* host_out);
int uc_precond_levels(uc_ctx* ctx, int64_t* shapes /* [levels][3] */);
/* Fraction of the owned stencil rows of (level, block) that are bitwise equal
 * to an interior row, so the apply kernels read that one shared row instead of
 * their own (synchronises). */
int uc_precond_uniform(uc_ctx* ctx, int level, int block, double* frac);

/* On-device initial conditions over the context's owned planes (SURVEY 8(f)
 * #4).  kind 0 = seed_initial_condition (free_growth.py:249-265), params
 * {anisotropy_strength, radius, far_temperature}; kind 1 =
 * directional_initial_condition (alloy.py:317-357), params {interface_x0,
 * amplitude, seed, smooth}.  extents[dim] are the mesh extents. */
int uc_initial_state(uc_ctx* ctx, int kind, const double* extents, const double* params,
                     double* out);

/* Per-step diagnostics of the time loop, replacing the host
 * passes of undercool/driver.py:186-229 over the new state:
 *   out[0] number of non-finite entries of unew      (driver.py:186)
 *   out[1] max |unew|                                (driver.py:187, BLOWUP_LIMIT)
 *   out[2..4] w@(T_new-T_old), w@(phi_new-phi_old), w@(phi_old-phi_prev)
 *          with w = mesh.integration_weights()       (_heat_balance, driver.py:86-98)
 *   out[5] composition integral at the new level     (_total_solute, driver.py:76-83)
 *   out[6..7] x_tip, found along the first node row  (extract_tip, diagnostics.py:69-89)
 * over the context's owned slab (`out` is a device array of UC_DIAG_N
 * doubles, zero where not requested; the tip only on the slab holding plane
 * 0).  Asynchronous on the context stream.  The group entry point exchanges
 * the ghost plane the composition integral needs and writes one out array per
 * slab; the caller adds the slab partials in slab order. */
#define UC_DIAG_BALANCE 1
#define UC_DIAG_SOLUTE 2
#define UC_DIAG_TIP 4
#define UC_DIAG_N 8
typedef struct uc_diag_args {
  int32_t what;                 /* UC_DIAG_* mask (non-finite and max are always computed) */
  int32_t pad;
  double elem_node_weight[8];   /* jxw @ values per local node (mesh.py:136) */
  double composition;           /* AlloyParams.composition (map_u_to_c, alloy.py:119-127) */
  double tip_level;             /* kernel.contour_level */
  double extent_x;              /* mesh.extents[0] (last linspace node) */
} uc_diag_args;
int uc_step_diagnostics(uc_ctx* ctx, const double* unew, const double* old,
                        const double* prev, const uc_diag_args* args, double* out);

/* map_u_to_c (alloy.py:119-127) of an owned block state into out[nloc] on the
 * device (numpy's operation order, no contraction). */
int uc_map_u_to_c(uc_ctx* ctx, const double* state, double composition, double* out);

/* Snapshot / mesh text writers (vtkio.py:31-86), host side:
 * byte-identical to the reference's files (numbers as Python repr prints
 * them).  counts/extents describe the mesh (dim entries); fields are HOST
 * arrays of n_nodes doubles in node order; format 0 = CSV
 * (write_snapshot_csv), 1 = legacy VTK structured grid (write_snapshot_vtk,
 * `comment` is its title line, "" = default).  `threads` host threads format
 * rows.  No GPU needed. */
int uc_write_snapshot(const char* path, int format, int dim, const int64_t* counts,
                      const double* extents, int nfields, const char* const* names,
                      const double* const* fields, const char* comment, int threads);
int uc_write_mesh_vtk(const char* path, int dim, const int64_t* counts, const double* extents,
                      int threads);
/* repr(float(x)) as a NUL-terminated string (out needs 32 bytes) */
int uc_repr_double(double x, char* out32);

/* FP64 issue-rate probe (DFMA chains over all SMs), for the FP64 roofline
 * denominator; synchronises.  Not part of the reference interface. */
int uc_fp64_probe(uc_ctx* ctx, int iters, double* ms_out, double* dfma_per_s);

/* Sticky status flags (synchronises); clear=1 resets them. */
int uc_status(uc_ctx* ctx, uc_status_t* out, int clear);

/* ---- Slab decomposition (paper §4 MPI subdomains) --------
 * Every *_group entry point takes the slabs driven by this process, ordered
 * by their slab_lo, with block vectors of the owned planes per slab.  Slab
 * neighbours are either local contexts (uc_ctx_link_local: same process and
 * device, planes copied on the stream — single-GPU emulation of k ranks) or
 * remote NCCL ranks (uc_comm_init_nccl + uc_ctx_set_neighbors: one process
 * per GPU, ncclSend/ncclRecv of one plane per field block, ncclAllReduce of
 * every dot product).  The single-context entry points above are the n = 1
 * case and are distributed automatically once a context has remote
 * neighbours. */
int uc_nccl_unique_id(const char* nccl_path, void* out128);
int uc_comm_init_nccl(const char* nccl_path, const void* id128, int rank, int nranks);
int uc_comm_finalize(void);
int uc_ctx_set_neighbors(uc_ctx* ctx, int lo_rank, int hi_rank);

/* Host-staged transport: the same remote branches of the exchange and global
 * sums (csrc/comm.cu) with the planes and partial sums staged through pinned
 * host buffers and moved by caller-supplied callbacks (e.g. torch.distributed
 * over gloo).  For testing the multi-rank code path where NCCL cannot run
 * (several ranks sharing one GPU); every call synchronises the stream.
 *   sendrecv: perform all ops (kind 0 = send `count` doubles from buf to peer,
 *             1 = receive into buf from peer) and return 0 on success;
 *   allreduce_sum: in-place sum of n doubles over all ranks, 0 on success. */
typedef struct uc_host_op {
  int32_t kind;
  int32_t peer;
  int64_t count;
  double* buf;
} uc_host_op;
typedef struct uc_host_transport {
  void* user;
  int (*sendrecv)(void* user, int nops, const uc_host_op* ops);
  int (*allreduce_sum)(void* user, double* vals, int n);
} uc_host_transport;
int uc_comm_init_host(const uc_host_transport* transport, int rank, int nranks);
int uc_ctx_link_local(uc_ctx* lower, uc_ctx* upper);

int uc_residual_group(uc_ctx* const* ctxs, int n, const uc_scheme* sc, int part,
                      const double* const* unew, const double* const* old,
                      const double* const* prev, const double* const* fixed,
                      double* const* out);
int uc_jv_group(uc_ctx* const* ctxs, int n, const uc_scheme* sc, const double* const* u,
                const double* const* fu, const double* const* v, double unorm,
                const double* const* old, const double* const* prev,
                const double* const* fixed, double* const* jv, double* eps_out);
/* global dot (b != NULL) or norm (b == NULL, do_sqrt = 1) over all slabs; synchronises */
int uc_dot_group(uc_ctx* const* ctxs, int n, const double* const* a, const double* const* b,
                 int do_sqrt, double* out);
/* basis: n x (k+2) device pointers (row per slab, slot k+1 is the output) */
int uc_arnoldi_group(uc_ctx* const* ctxs, int n, const double* const* basis, int k,
                     double* const* w, double scale, double* h_host, int* broke);
int uc_precond_build_group(uc_ctx* const* ctxs, int n, const uc_scheme* sc,
                           const double* const* states, const uc_precond_cfg* cfg);
int uc_precond_apply_group(uc_ctx* const* ctxs, int n, const double* const* v,
                           double* const* out);
int uc_step_diagnostics_group(uc_ctx* const* ctxs, int n, const double* const* unew,
                              const double* const* old, const double* const* prev,
                              const uc_diag_args* args, double* const* out);

#ifdef __cplusplus
}
#endif
#endif /* UC_B200_H */

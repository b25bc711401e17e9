/*
 * mhdg.h -- C ABI of the B200 (sm_100a) macro-element HDG hot path.
 *
 * Plain pointers and sizes only (no torch types).  Every pointer inside the
 * structs and every array argument is a DEVICE pointer (FP64 unless noted,
 * int32 for index tables); `stream` is a cudaStream_t passed as void*.
 * All calls are stream-ordered and asynchronous unless documented otherwise.
 *
 * Each entry point replaces one reference operation (paths relative to
 * /root/reference/pkg/src/macrohdg/):
 *
 *   mhdg_assemble           assembly.py:339-618  assemble_system
 *                           (residual(): assembly.py:621, jacobian(): :626)
 *   mhdg_condense           condense.py:62-70 + 130-158
 *                           CondensedSchur.build (_schur_correction + inv;
 *                           here: Schur GEMM + batched LU, partial pivoting)
 *   mhdg_apply_trace        condense.py:91-103  CondensedSchur.apply_trace
 *   mhdg_condensed_rhs      condense.py:105-110 CondensedSchur.rhs
 *   mhdg_recover            condense.py:112-127 CondensedSchur.recover
 *   mhdg_gradient_refresh   assembly.py:247-252 Discretization.gradient_refresh
 *   mhdg_precond_build      krylov.py:194-232   block_precond_build
 *   mhdg_precond_apply      krylov.py:234-236   (closure returned by it)
 *   mhdg_face_reduce        condense.py:48-51   _scatter_add (deterministic)
 *   mhdg_*_window           the same operations on a window of macros whose blocks
 *                           were just re-formed from (u, q, uhat): the paper's "store
 *                           only S^-1 and transformation data" variant,
 *                           condense.py:62-127 without resident LocalBlocks
 *
 * Layouts are the reference's (assembly.py:6-8): volume dof node*ns+s,
 * gradient dof (l*L+node)*ns+s, trace dof (f*Lf+g)*ns+s, local trace
 * (mac, lf, g, s).  Blocks use the LocalBlocks shapes of assembly.py:293-312.
 *
 * Diagnostic A/B knobs (kernel variants for cross-checks) are not part of
 * this ABI; they live in paper_2402_11361_b200/csrc/mhdg_tuning.h.
 *
 * Errors: the return value is MHDG_OK or MHDG_ERR_CUDA (launch failure).
 * Data-dependent failures are reported through the device status word
 * `status` (mhdg_status, int32[4]): code, macro/face index, component, and
 * the value bits are written by the first failing thread; the host reads it
 * after the call and maps it to the reference exception classes
 * (AdmissibilityError physics.py:23, FactorizationError condense.py:40,
 * PreconditionerError krylov.py:47).
 */
#ifndef MHDG_H
#define MHDG_H

#ifdef __cplusplus
extern "C" {
#endif

#define MHDG_OK 0
#define MHDG_ERR_ADMISSIBILITY 1
#define MHDG_ERR_FACTORIZATION 2
#define MHDG_ERR_PRECONDITIONER 3
#define MHDG_ERR_CONFIG 4
#define MHDG_ERR_CUDA 5

/* discretization: reference tables, geometry, layouts (device pointers) */
typedef struct {
  int dim, ns, nf;            /* d, d+2, d+1 */
  int n_mac, n_faces, n_trace;
  int L, Lf;                  /* volume / face lattice sizes */
  int n_sub, nloc, nq;        /* sub-elements, nodes per sub, volume qp per sub */
  int n_tri, nlocf, nqf;      /* face sub-elements, nodes per face sub, qp per face sub */
  double face_fac;            /* (d-1)!: face weight = w_face_ref * face_fac * area */
  /* reference tables */
  const double *mass;         /* L*L */
  const double *mass_inv;     /* L*L */
  const double *minv_d;       /* d*L*L   M^-1 D[r] */
  const double *weak_deriv;   /* d*L*L   D[r][i][j] = int phi_j d_r phi_i (basis.py:412-424) */
  const double *gf;           /* nf*L*Lf  M^-1[:, fvn[f]] face_mass */
  const double *face_mass;    /* Lf*Lf */
  const int *face_vol_nodes;  /* nf*Lf */
  const int *sub_conn;        /* n_sub*nloc */
  const double *phi_vol;      /* nq*nloc */
  const double *grad_ref;     /* n_sub*nq*nloc*d */
  const double *w_ref;        /* n_sub*nq */
  const int *tri_conn;        /* n_tri*nlocf */
  const double *phi_face;     /* nqf*nlocf */
  const double *w_face_ref;   /* n_tri*nqf */
  const double *pm_vol;       /* n_sub*nq*d*L : sum_b phi[q,b] minv_d[r][conn[K,b], :] */
  const double *pm_face;      /* nf*n_tri*nqf*d*L */
  /* inverse incidence (CSR) for deterministic gathers */
  const int *vn_ptr, *vn_sub;  /* L+1 ; entries K*nloc+a with sub_conn[K,a] = node */
  const int *vf_ptr, *vf_ent;  /* L+1 ; entries f*Lf+g with face_vol_nodes[f,g] = node */
  const int *fn_ptr, *fn_ent;  /* Lf+1 ; entries T*nlocf+a with tri_conn[T,a] = g */
  /* geometry per macro */
  const double *det;          /* n_mac */
  const double *inv_jac;      /* n_mac*d*d */
  const double *normals;      /* n_mac*nf*d */
  const double *areas;        /* n_mac*nf */
  const double *h_sub;        /* n_mac*n_sub */
  const int *gather;          /* n_mac*nf*Lf*ns  global trace dof of each local dof */
  const int *scatter_src;     /* n_trace*2  local flat indices summed per dof, -1 = none */
  /* boundary data */
  const int *bc_kind;         /* n_mac*nf  0 interior, 1 Dirichlet, 2 wall */
  const double *wall_e;       /* n_mac*nf */
  const double *wall_u;       /* n_mac*nf*d */
  const double *u_dir;        /* n_mac*nf*n_tri*nqf*ns */
  const double *source;       /* n_mac*n_sub*nq*ns or NULL */
  /* face skeleton for the block preconditioner */
  const int *face_macros;     /* n_faces*2 (-1 = none) */
  const int *face_locals;     /* n_faces*2 */
  /* volume nodes lying on the macro boundary (ascending) */
  int n_face_nodes;
  const int *node_to_face;    /* L: index into the face-node list, -1 for interior nodes */
  const double *minv_d_face;  /* d*n_face_nodes*L: rows of M^-1 D_r at the face nodes */
  /* distinct grad_ref[K] tables (sub-elements of one orientation class share
     them: 2 classes in 2D, <= 6 in 3D) */
  int n_grad_cls;
  const double *grad_cls;     /* n_grad_cls*nq*nloc*d */
  const int *grad_cls_of;     /* n_sub: class of each sub-element */
} mhdg_disc;

typedef struct {
  double gamma, prandtl, re_acoustic, mach_ref, mu, re_flow;
} mhdg_flow;

typedef struct {
  double dt_coeff;      /* d_ii/dt, 0 when steady */
  const double *hist;   /* n_mac*L*ns or NULL */
  double pseudo_dt;     /* +inf: none */
  double supg_dt;       /* +inf: none */
} mhdg_stage;

typedef struct {
  double *state_state;       /* n_mac*(L ns)^2 */
  double *face_state_trace;  /* n_mac*nf*(Lf ns)^2 */
  double *face_trace_state;
  double *face_trace_trace;
  double *wdgdq_vol;         /* n_mac*n_sub*nq*d*d*ns*ns */
  double *wdgdq_face;        /* n_mac*nf*(n_tri nqf)*d*ns*ns */
  double *trace_face_scale;  /* n_mac*nf */
} mhdg_blocks;

typedef struct {
  double *supg_tau;          /* n_mac*n_sub*nq */
  double *supg_jac;          /* n_mac*n_sub*nq*d*ns*ns */
  double *face_stab;         /* n_mac*nf*(n_tri nqf)*ns*ns */
  double *face_visc_state;   /* n_mac*nf*(n_tri nqf)*ns */
} mhdg_frozen;

/* condensed operator S = A_uu - A_uq A_qq^-1 A_qu (n = L*ns), factored per
   macro into `lu` (mhdg_packed_lu_size(n) doubles per macro) according to
   `kind`:
     kind 1 (default): LU with partial pivoting (the rows never move; perm[k]
       = physical row of logical pivot k), packed in block-triangular solve
       order (csrc/packed_lu.cuh): per 64-row block the L panel and inv(L_bb)
       for the forward sweep, then the U panel and inv(U_bb) for the backward
       sweep, column-major inside panels and triangles;
     kind 0: the explicit inverse S^-1 (what the reference's np.linalg.inv
       stores, condense.py:67) by Gauss-Jordan with partial pivoting, in the
       tiled order of csrc/tiled_inv.cuh (64-row blocks of 32-column tiles).
   `scratch` (n_mac*n*n, or scratch_macros*n*n) holds S before factorization.  `work`
   (mhdg_apply_work_size doubles, or NULL) holds the per-macro hand-off
   vectors of the split apply (pre -> factor solve -> post); with NULL the
   fused single-kernel apply runs. */
typedef struct {
  double *lu;                /* n_mac*mhdg_packed_lu_size(n) */
  int *perm;                 /* n_mac*n */
  double *scratch;           /* n_mac*n*n */
  double *work;              /* mhdg_apply_work_size(disc) or NULL */
  int kind;                  /* 0: explicit S^-1, tiled (csrc/tiled_inv.cuh), Gauss-Jordan;
                                1: packed LU (csrc/packed_lu.cuh), perm = pivot rows */
  int scratch_macros;        /* macros `scratch` holds: <= 0 or >= n_mac: all (n_mac*n*n);
                                else mhdg_condense forms and factors S that many macros at a
                                time (memory-lean: C5's (m, p) = (2, 3) slabs) */
} mhdg_factors;

/* Largest local Schur size n = L*ns the factor kernels take for factor `kind`
   (mhdg_factors.kind); mhdg_condense returns MHDG_ERR_CONFIG above it. */
int mhdg_factor_max_n(int kind);

/* doubles of mhdg_factors.work for this discretization */
long long mhdg_apply_work_size(const mhdg_disc *disc);

/* One ICGS Arnoldi orthogonalisation (krylov.py:51-58): with V_j = rows 0..j of
   V (row stride ldv), h = V_j w; w -= V_j^T h; h2 = V_j w; w -= V_j^T h2;
   out[0..j] = h + h2, out[j+1] = ||w|| (w updated in place).  Three fused
   streaming passes over V_j (mhdg_vec_pass modes 0, 1, 2), any n,
   deterministic reductions (the result depends on n only); j <= 62.
   scratch: mhdg_icgs_scratch_size(n) doubles, zeroed once before first use
   (the passes leave their completion ticket re-armed). */
int mhdg_icgs(int n, int j, const double *V, long long ldv, double *w, double *out, double *scratch,
              void *stream);
long long mhdg_icgs_scratch_size(int n);

/* One streaming pass of the Krylov vector algebra over rows 0..rows-1 of V
   (row stride ldv; rows <= 64) and the n-vector w, deterministic:
     mode 0: out[i] = V_i . w                        (the dots of krylov.py:53, 55)
     mode 1: w -= sum_i coef[i] V_i; out[i] = V_i . w (ICGS update + re-orthogonalisation dots)
     mode 2: w -= sum_i coef[i] V_i; out[0] = w . w
     mode 3: w += sum_i coef[i] V_i                  (x + V^T y, krylov.py:121-122, 188-189)
     mode 4: out[0] = w . w                          (squared norms, krylov.py:72-168)
   Sums are this device's partial sums (a distributed caller allreduces `out`);
   coef and out are device arrays.  scratch as for mhdg_icgs. */
int mhdg_vec_pass(long long n, int rows, const double *V, long long ldv, double *w, const double *coef, int mode,
                  double *out, double *scratch, void *stream);

/* Per-kernel timeline: while enabled, the library records a CUDA event pair
   around each of its kernels on the caller's stream (capacity = max records).
   mhdg_timeline_end synchronises, disables recording and returns, per slot,
   the summed milliseconds and the record counts (16 slots: 0 apply pre,
   1 apply factor solve, 2 apply post, 3 fused apply, 4 generic apply, 5 face
   reduce, 6 Schur complement, 7 factorization, 8 factor packing, 9 assembly,
   10 stored-operator apply, 11 ICGS, 12 preconditioner build, 13
   preconditioner apply, 14 halo pack/unpack). */
int mhdg_timeline_begin(int capacity);
int mhdg_timeline_end(double *ms, int *counts);

/* doubles per macro of the factor buffer (either kind) */
long long mhdg_packed_lu_size(int n);

/* Residuals (and, with want_jac, blocks + frozen coefficients).
   frozen_in != NULL evaluates the residual with frozen coefficients (the
   finite-difference oracle mode of assembly.py:84-96).
   R_trace_loc: n_mac*nf*Lf*ns scratch; R_trace = its deterministic face sum. */
int mhdg_assemble(const mhdg_disc *disc, const mhdg_flow *flow, const mhdg_stage *stage,
                  const double *u, const double *q, const double *uhat,
                  double *R_grad, double *R_state, double *R_trace_loc, double *R_trace,
                  int want_jac, const mhdg_blocks *blocks, const mhdg_frozen *frozen_out,
                  const mhdg_frozen *frozen_in, int *status, void *stream);

/* S = state_state - A_uq A_qq^-1 A_qu, then in-place batched LU with partial pivoting. */
int mhdg_condense(const mhdg_disc *disc, const mhdg_blocks *blocks, const mhdg_factors *fac,
                  int *status, void *stream);

/* Schur complement only (no factorization), into fac->scratch (n x n per macro). */
int mhdg_schur_matrix(const mhdg_disc *disc, const mhdg_blocks *blocks, const mhdg_factors *fac,
                      void *stream);

/* LU-factor the n x n matrices in fac->scratch in place (partial pivoting) and pack into fac->lu. */
int mhdg_lu_factor(const mhdg_disc *disc, const mhdg_factors *fac, int *status, void *stream);

/* y_mac = S^-1 b_mac for all macros (b, y: n_mac*n; may alias). */
int mhdg_lu_solve(const mhdg_disc *disc, const mhdg_factors *fac, const double *b, double *y,
                  void *stream);

/* y = A_hat x (global trace vectors, n_trace).  y_loc: n_mac*nf*Lf*ns scratch. */
int mhdg_apply_trace(const mhdg_disc *disc, const mhdg_blocks *blocks, const mhdg_factors *fac,
                     const double *x, double *y, double *y_loc, void *stream);

/* Local (unscattered) part of the apply, y_loc only. */
int mhdg_apply_trace_local(const mhdg_disc *disc, const mhdg_blocks *blocks,
                           const mhdg_factors *fac, const double *x, double *y_loc, void *stream);

/* Stored local trace operators (B_A representation, csrc/ahat.cu): A^T[m][k][:] = column k
 * of macro m's condensed trace block (the apply of the unit local trace e_k), for
 * k < nf*Lf*ns; the blocks the reference's dense_trace_operator assembles
 * (condense.py:269-290).  at: n_mac*ltr*ltr; x_loc, y_loc: n_mac*ltr scratch; ident:
 * n_mac*ltr ints of scratch.  Runs ltr local applies. */
int mhdg_ahat_form(const mhdg_disc *disc, const mhdg_blocks *blocks, const mhdg_factors *fac,
                   double *at, double *x_loc, double *y_loc, int *ident, void *stream);

/* y = A_hat x from the stored blocks (replaces CondensedSchur.apply_trace,
 * condense.py:91-103): batched GEMV + face reduction.  y_loc: n_mac*ltr scratch. */
int mhdg_ahat_apply(const mhdg_disc *disc, const double *at, const double *x, double *y,
                    double *y_loc, void *stream);
int mhdg_ahat_apply_local(const mhdg_disc *disc, const double *at, const double *x,
                          double *y_loc, void *stream);

/* mhdg_apply_trace_local for the contiguous macro range [mac0, mac0 + count) only
   (y_loc entries of the other macros untouched): a slab applies its interior
   macros while the forward halo is in flight and the macros next to ghost faces
   after it arrives (multi-GPU). */
int mhdg_apply_trace_local_range(const mhdg_disc *disc, const mhdg_blocks *blocks, const mhdg_factors *fac,
                                 const double *x, double *y_loc, int mac0, int count, void *stream);

/* Halo messages of the slab decomposition: buf[i] = src[idx[i]] (pack), and
   dst[idx[i]] = buf[i] or, with accumulate, dst[idx[i]] += buf[i] (unpack;
   idx entries unique), i < n. */
int mhdg_halo_gather(long long n, const int *idx, const double *src, double *buf, void *stream);
int mhdg_halo_scatter(long long n, const int *idx, const double *buf, double *dst, int accumulate, void *stream);

/* Face sum of the first n_out trace dofs with the reverse halo folded in: y[i] =
   y_loc[src0] + (y_loc[src1] if the dof has a second local side, else
   remote[remote_src[i]] if remote_src[i] >= 0, else 0) -- the other rank's side of
   a face split across slabs (condense.py:48-51 across ranks). */
int mhdg_face_reduce_remote(const mhdg_disc *disc, const double *y_loc, const int *remote_src, const double *remote,
                            int n_out, double *y, void *stream);

/* y[dof] = sum of the (one or two) local contributions, in flat-index order. */
int mhdg_face_reduce(const mhdg_disc *disc, const double *y_loc, double *y, void *stream);

/* b = -R_trace + scatter(A_hu S^-1 (R_U - A_uq A_qq^-1 R_Q) ... ) (condense.py:105-110). */
int mhdg_condensed_rhs(const mhdg_disc *disc, const mhdg_blocks *blocks, const mhdg_factors *fac,
                       const double *R_grad, const double *R_state, const double *R_trace,
                       double *b, double *b_loc, void *stream);

/* (du, dq) from the trace update (condense.py:112-127). */
int mhdg_recover(const mhdg_disc *disc, const mhdg_blocks *blocks, const mhdg_factors *fac,
                 const double *R_grad, const double *R_state, const double *dtrace,
                 double *du, double *dq, void *stream);

/* q = A_qq^-1 (-A_qu u - A_qh uhat) (assembly.py:247-252). */
int mhdg_gradient_refresh(const mhdg_disc *disc, const double *u, const double *uhat, double *q,
                          void *stream);

/* Per-face B_f = sym(sum_sides P^T face_trace_trace P), Cholesky, explicit
   inverse (krylov.py:194-232).  inv: n_faces*bs*bs, bs = Lf*ns. */
int mhdg_precond_build(const mhdg_disc *disc, const mhdg_blocks *blocks, double *inv, int *status,
                       void *stream);

/* As mhdg_precond_build, adding extra[f] (n_faces*bs*bs, canonical face order, or
   NULL) to each face block before symmetrising: the contribution of a face side
   that lives on another rank (multi-GPU slabs).  Build and apply cover faces
   [0, disc->n_faces) only, so a slab passes a copy of its disc with n_faces set
   to its owned-face count (owned faces come first; ghost faces carry one side
   and are never factorised). */
int mhdg_precond_build_ext(const mhdg_disc *disc, const mhdg_blocks *blocks, const double *extra, double *inv,
                           int *status, void *stream);

/* out[i] = P^T face_trace_trace[macs[i], lfs[i]] P (bs x bs, the face's canonical
   node order): one side's share of the block preconditioner, for export. */
int mhdg_side_blocks(const mhdg_disc *disc, const mhdg_blocks *blocks, const int *macs, const int *lfs, int count,
                     double *out, void *stream);

/* y = blockdiag(inv) v (krylov.py:234-236). */
int mhdg_precond_apply(const mhdg_disc *disc, const double *inv, const double *v, double *y,
                       void *stream);

/* ---- Coupling-recompute representation (B_min: "store only
   S^-1 and transformation data").  Only the S factors (and the face preconditioner) stay
   resident; the coupling blocks the trace operator needs (condense.py:91-127) are re-formed
   from the linearisation state (u, q, uhat) one window of macros at a time.  In every call
   `blocks_w` (and `frozen_w`, R_*_w) hold the window [mac0, mac0 + count) only, while the
   factors and all other vectors are whole-mesh arrays; fac->scratch must hold at least
   `count` macros (n*n doubles each). ---- */

/* mhdg_assemble restricted to the window.  want_jac: 0 residuals only, 1 residuals +
   blocks + frozen coefficients, 2 couplings only (face blocks, dG/dq stashes and
   trace_face_scale; no state_state, no frozen output, no residual vectors: R_*_w and
   frozen_w may be NULL).  No R_trace face sum (call mhdg_face_reduce on whole-mesh data).
   Status macro indices are window-relative. */
int mhdg_assemble_window(const mhdg_disc *disc, const mhdg_flow *flow, const mhdg_stage *stage,
                         const double *u, const double *q, const double *uhat,
                         double *R_grad_w, double *R_state_w, double *R_trace_loc_w, int want_jac,
                         const mhdg_blocks *blocks_w, const mhdg_frozen *frozen_w, int mac0, int count,
                         int *status, void *stream);

/* mhdg_condense for the window's macros: S from blocks_w, factors written at their
   whole-mesh positions. */
int mhdg_condense_window(const mhdg_disc *disc, const mhdg_blocks *blocks_w, const mhdg_factors *fac,
                         int mac0, int count, int *status, void *stream);

/* mhdg_apply_trace_local for the window (y_loc: whole-mesh array, the window's part written). */
int mhdg_apply_trace_local_window(const mhdg_disc *disc, const mhdg_blocks *blocks_w, const mhdg_factors *fac,
                                  const double *x, double *y_loc, int mac0, int count, void *stream);

/* Local part of mhdg_condensed_rhs for the window (R_grad, R_state, b_loc whole-mesh);
   finish with mhdg_face_reduce_axpy(b_loc, R_trace, -1). */
int mhdg_condensed_rhs_local_window(const mhdg_disc *disc, const mhdg_blocks *blocks_w, const mhdg_factors *fac,
                                    const double *R_grad, const double *R_state, double *b_loc,
                                    int mac0, int count, void *stream);

/* mhdg_recover for the window (all vectors whole-mesh). */
int mhdg_recover_window(const mhdg_disc *disc, const mhdg_blocks *blocks_w, const mhdg_factors *fac,
                        const double *R_grad, const double *R_state, const double *dtrace,
                        double *du, double *dq, int mac0, int count, void *stream);

/* sums[f] += P^T face_trace_trace P of the window's sides of every face f (sums:
   n_faces*bs*bs, zeroed before the first window; windows in ascending order give the
   bitwise sum mhdg_precond_build forms), then mhdg_precond_build_sums inverts them. */
int mhdg_face_sum_window(const mhdg_disc *disc, const mhdg_blocks *blocks_w, double *sums, int mac0, int count,
                         void *stream);
int mhdg_precond_build_sums(const mhdg_disc *disc, const double *sums, double *inv, int *status, void *stream);

/* y[dof] = face sum of y_loc (as mhdg_face_reduce) + alpha * add[dof] (add may be NULL). */
int mhdg_face_reduce_axpy(const mhdg_disc *disc, const double *y_loc, const double *add, double alpha,
                          double *y, void *stream);

/* number of kernel launches issued by this library since load (diagnostics) */
long long mhdg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MHDG_H */

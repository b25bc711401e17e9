/*
 * mhdg_tuning.h -- diagnostic and A/B-measurement knobs of libmhdg.so.
 *
 * NOT part of the drop-in C ABI (include/mhdg.h): a reference-side binding
 * never calls these.  They select between kernel variants for cross-checks in
 * the tests and for the A/B measurements under tools/; every knob is
 * process-global and defaults to the production path.  Set them only while no
 * other thread is issuing library calls.
 */
#ifndef MHDG_TUNING_H
#define MHDG_TUNING_H

#ifdef __cplusplus
extern "C" {
#endif

/* Schur-complement kernel: 0 (default) the stage-pipelined FP64 tensor-core kernel
   (schur.cu) when its stages fit, otherwise the per-macro FFMA kernel. */
void mhdg_set_schur_variant(int v);

/* Panel width of k_lu4: 32 (default; 192 threads, two CTAs per SM) or 64 (one CTA
   per SM; threads 256 or 384). */
void mhdg_set_lu_panel(int nb, int threads);

/* L2 priority of k_lu4's trailing-update traffic: evict_last on the macros with
   mac % mode != 0 (mode >= 2; default 2 = every other macro), on all (1) or none (0). */
void mhdg_set_lu_l2mode(int mode);

/* Persistent grid of k_lu4: ctas > 0 launches that many CTAs walking the macros
   (fewer trailing matrices resident at once); 0 (default): one CTA per macro. */
void mhdg_set_lu_grid(int ctas);

/* LU kernel shape for n <= 192: 2 (default) CTAs of 32 / 64 / 64 threads for n <= 64 / 128 / 192
   (2 / 2 / 3 rows per thread, 8 / 6 / 4 CTAs per SM); 1: as 2 but 96 threads for n <= 192;
   0: the 192-thread, two-CTAs-per-SM kernel. */
void mhdg_set_lu_small(int on);

/* 1 (default): split apply (pre / factor solve / post kernels) when `work` is set;
   0: fused single-kernel apply. */
void mhdg_set_apply_split(int on);

/* 1 (default): the compile-time specialised TMA-streamed apply kernels when one
   matches (dim, m, p); 0: always the generic kernel. */
void mhdg_set_stream_enabled(int on);

/* L2 prefetch lookahead of the streamed apply in pieces: default 4; 0 = the
   shared-memory ring only. */
void mhdg_set_stream_prefetch(int pieces);

/* Face-block preconditioner build: 0 (default) the register-tile Gauss-Jordan sweep for
   face blocks up to 144 dofs; 1: the shared-memory Cholesky + triangular inverse. */
void mhdg_set_precond_variant(int v);

/* Couplings-only assembly (mhdg_assemble_window, want_jac = 2): 1 (default) the dedicated
   k_couplings kernel; 0: k_assemble's Jacobian path with the state_state work skipped. */
void mhdg_set_couplings_kernel(int on);

/* CTAs per launch of the last streamed pre/post kernel (diagnostics). */
int mhdg_stream_grid(void);

#ifdef __cplusplus
}
#endif
#endif /* MHDG_TUNING_H */

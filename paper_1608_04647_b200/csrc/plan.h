// Device-side view of an SRM plan (passed by value to every kernel) and the
// kernel launchers of smallmat.cu.  Internal; not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace srm {

// per local subject record in DevPlan::subj (int64 x kSubjCols)
enum SubjCol {
  SC_ROW_OFF = 0,   // first row in the concatenated X-hat / A / W arrays
  SC_V = 1,         // voxel count
  SC_CHUNK0 = 2,    // first V-chunk index (partials)
  SC_NCHUNK = 3,    // number of V-chunks
  SC_GLOBAL = 4,    // global subject index (srm.py:237 rank_offsets)
  SC_SLOT = 5,      // record slot in the E-step term table
  kSubjCols = 8
};

// scalar fields at the end of each E-step term record (after kp * ldx doubles)
enum RecCol { RC_RHO2 = 0, RC_V = 1, RC_SQNORM = 2, kRecScalars = 8 };

// scalar fields after the kp * ldx reduced sum in RED / REDLOCAL
enum RedCol { RD_RHO0 = 0, RD_VLOGRHO = 1, RD_SQRHO = 2, RD_VSUM = 3, kRedScalars = 8 };

// tail scratch scalars
enum TailCol { TS_LOGDET_SIGMA = 0, TS_LOGDET_PREC = 1, TS_TRACE = 2, kTailScalars = 8 };

// column tile width of apply_m (W^T Xhat = M^T B): 128, or 64 for kp > 112
// (DevPlan::apply_cols, ntile_apply = ceil(ldx / apply_cols))
inline int apply_cols_for(int64_t kp) { return kp > 112 ? 64 : 128; }
// TR chunk of gram_from_b (A^T A = B S^T / 2)
constexpr int kGfbCols = 128;

struct DevPlan {
  int n_local, n_total, n_order;
  int sub0, nsub;  // subject window [sub0, sub0 + nsub) of the per-subject kernels (default: all)
  int flags;
  int xf32;  // X-hat stored in fp32 (per-iteration polar may run in fp32; the final one is exact)
  int64_t T, K, ldx, kp, ldo;
  int ntile_apply;  // apply_cols-column tiles of ldx
  int apply_cols;   // apply_m column tile (apply_cols_for(kp))
  int ntile_tail;   // 32-column tiles of ldx
  int polar_cross;  // the M-step polar (k_ns_polar / k_ns_polar_g) writes the cross term into crossp
  int64_t term_stride, red_stride, hist_stride;
  // regions
  void* xhat;
  double* amat;
  double* wout;
  double* mu;
  double* rowsq;
  unsigned long long* cmax;  // [n_local][ldx] max |Xhat[:, t]| as IEEE bits (int8 Gram path; else null)
  double* terms;
  double* red;
  double* redlocal;
  double* S;
  double* sigma;
  double* sinv;      // [kp][kp] -Sigma_s^{-1} of the coming E-step (k_tail_inv)
  double* var;
  double* cmat;
  double* tailscr;
  double* sspart;    // [ntile_tail][kp][kp]
  double* tailpart;  // [ntile_tail][4]
  double* part;      // [chunks][kp][ldo]
  double* bred;      // [n_local][kp][ldo]
  double* gfb_part;  // [n_local][gfb_chunks][kp][kp] partial A^T A = B S^T / 2 per TR chunk
  int32_t* gfb_count;  // [n_local] CTAs done per subject (reset by the last one)
  int gfb_chunks;      // kGfbCols-column chunks of ldx
  double* mmat;      // [n_local][kp][kp]
  double* qmat;      // [n_local][kp][kp]
  double* qscr;      // [n_local][kp][kp]
  double* crossp;    // [n_local][ntile_apply]
  double* scal;      // [n_local][8]: {jacobi sweeps, ...}
  double* nsg;       // [n_local][4][kp][kp]: Newton-Schulz matrices of the kp > 80 transform (else null)
  double* st;        // [ldx][kp]: S^T (Gram path operand)
  double* gram;      // [n_local][ldx][ldx]: X_i^T X_i (Gram path)
  float* af;         // [rows][np]: A_i in fp32 (tensor-core path)
  float* sf;         // [2][np][ldx]: S split into tf32 hi / lo (tensor-core path)
  int np;            // tensor-core feature padding (multiple of 16)
  double* hist;      // [iterations][hist_stride]
  int32_t* status;
  int32_t* iter;          // device iteration counter (one graph serves every iteration)
  int n_hist;             // history rows
  const int64_t* subj;   // [n_local][kSubjCols]
  const int32_t* order;  // [n_order] record slots, ascending global subject index
  // SRM_FLAG_COLBLOCK exchange: world column blocks of xw TRs; block records
  // of xrec = kp * xw + kRecScalars doubles, reduced blocks of xred
  int world, rank, max_local, xw;
  int64_t xrec, xred;
  double* xsend;            // [world][max_local][xrec]
  double* xrecv;            // [world][max_local][xrec]
  double* xredbuf;          // [world][xred]
  const int32_t* xcounts;   // [world] subjects per rank
};

cudaError_t launch_prep(const DevPlan& p, int local, int64_t V, const void* x, int x_dtype,
                        int64_t ld, int xhat_dtype, cudaStream_t s);
cudaError_t launch_subject_sqnorm(const DevPlan& p, cudaStream_t s);
cudaError_t launch_reduce_chunks(const DevPlan& p, cudaStream_t s);
cudaError_t launch_eig_polar(const DevPlan& p, int init, cudaStream_t s);
cudaError_t launch_apply_m(const DevPlan& p, int with_cross, cudaStream_t s);
// A_i^T A_i = B_i S^T / 2 into the K x K block of every subject's reduced
// record (bred[i][:, ldx:ldx+kp]), split over TR chunks
cudaError_t launch_gram_from_b(const DevPlan& p, cudaStream_t s);
cudaError_t launch_finalize_rho(const DevPlan& p, int init, cudaStream_t s);
// finalize_rho of an iteration plus the iteration-counter advance, one block
// (when nsub <= 1024)
bool finalize_rho_advances(const DevPlan& p);
cudaError_t launch_finalize_rho_advance(const DevPlan& p, cudaStream_t s);
cudaError_t launch_set_iteration(const DevPlan& p, int iteration, int advance, cudaStream_t s);
cudaError_t launch_reduce_terms(const DevPlan& p, double* dst, const int32_t* order, int count,
                                cudaStream_t s, bool ident = false);
cudaError_t launch_tail(const DevPlan& p, cudaStream_t s);
// SRM_FLAG_COLBLOCK exchange kernels (smallmat.cu)
cudaError_t launch_xchg_pack(const DevPlan& p, cudaStream_t s);
cudaError_t launch_xchg_reduce(const DevPlan& p, cudaStream_t s);
cudaError_t launch_xchg_unpack(const DevPlan& p, cudaStream_t s);
cudaError_t launch_tail_inv(const DevPlan& p, cudaStream_t s);
cudaError_t launch_tail_kk(const DevPlan& p, cudaStream_t s);
cudaError_t launch_tail_s(const DevPlan& p, cudaStream_t s);
cudaError_t launch_tail_sigma(const DevPlan& p, cudaStream_t s);
cudaError_t launch_mirror_gram(const DevPlan& p, int first, int count, cudaStream_t s);
// int8-sliced Gram (ozaki.cu): exponents and slices of local subjects
// [first, first + count) (the column maxima come from the demean pass)
cudaError_t launch_oz_prepare(const DevPlan& p, int x_dtype, int nsl, int first, int count,
                              unsigned long long* cmax, int8_t* q, int64_t lq, int32_t* expo, int64_t max_v,
                              cudaStream_t st);
// slices of the init draw G (AMAT) of local subjects [first, first + count):
// column maxima, exponents and seven-slice records [i][k][vb] (pitch lqg)
cudaError_t launch_oz_init_slices(const DevPlan& p, int first, int count, int8_t* qg, int64_t lqg, int32_t* expog,
                                  unsigned long long* cmaxg, int64_t max_v, cudaStream_t st);
cudaError_t launch_reset(const DevPlan& p, cudaStream_t s);
cudaError_t launch_apply_w(const DevPlan& p, const void* items_a, int n_items, cudaStream_t s);
cudaError_t launch_apply_w_f32(const DevPlan& p, const void* items_a, int n_items, cudaStream_t s);

// stateless helpers
cudaError_t launch_spd_inverse(double* a, int n, int32_t* status, cudaStream_t s);
cudaError_t launch_polar_small(const double* gram, int64_t ldg, int n, double* m, int64_t ldm,
                               int32_t* status, cudaStream_t s);
cudaError_t launch_apply_right(const double* a, int64_t lda, int64_t v, int k, const double* m,
                               int64_t ldm, double* w, int64_t ldw, cudaStream_t s);

int max_supported_k();
bool ns_polar_supported(int kp);
cudaError_t launch_ns_polar(const DevPlan& p, int init, cudaStream_t s);
bool ns_polar_f32_supported(int kp);
// fp64 polar from the fp32 Newton-Schulz M (80 < kp <= 112); scal[i][1] = 1 where it converged,
// with `warn` a subject it leaves raises SRM_WARN_POLAR_CONDITION
cudaError_t launch_ns_refine(const DevPlan& p, cudaStream_t s, int warn = 0);
cudaError_t launch_final_polar(const DevPlan& p, cudaStream_t s);
cudaError_t launch_ns_polar_f32(const DevPlan& p, int init, cudaStream_t s);
// fp64 Newton-Schulz for 80 < kp <= 128 with its matrices in DevPlan::nsg
bool ns_polar_g_supported(int kp);
cudaError_t launch_ns_polar_g(const DevPlan& p, int init, cudaStream_t s);
cudaError_t launch_eig_polar_exact(const DevPlan& p, int init, cudaStream_t s);

}  // namespace srm

// Internal launcher interface between the C-ABI layer (capi.cu) and the
// kernel translation units.  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace srm {

// One CTA of the V-contraction kernel: out[m][n0+j] += sum_{c<rows} L[c][m] R[c][n0+j]
// for m < KP, j < ncols (<= 128).  Offsets are in elements of each base.
struct ItemE {
  int64_t l_off;  // L(row 0, col 0) of this chunk
  int64_t r_off;  // R(row 0, col n0)
  int64_t o_off;  // out(0, n0)
  int32_t rows;   // contraction rows in this chunk
  int32_t ncols;  // valid output columns (<= 128)
  int32_t mrows;  // valid output rows (<= KP)
  int32_t pad;
};

// One CTA of the T-contraction kernel: out[r][f] = alpha sum_t X[r][t] S[f][t]
// for r < rows (<= 128), f < KP, t < ldx.
struct ItemA {
  int64_t x_off;  // X(row r0, 0)
  int64_t o_off;  // out(row r0, 0)
  int32_t rows;   // valid rows (<= 128)
  int32_t pad;
};

// V-contraction; L and R are f64 or f32 (X-hat), (f32, f64) is not instantiated.
cudaError_t launch_contract_e(int kp, int l_dtype, int r_dtype, const void* L, int64_t ldl, const void* R,
                              int64_t ldr, double* out, int64_t ldo, double alpha,
                              const ItemE* items, int n_items, cudaStream_t stream);

// T-contraction over `ncontract` columns (multiple of 16).
cudaError_t launch_contract_a(int kp, int x_dtype, const void* X, int64_t ldx, const double* S,
                              int64_t lds, int64_t ncontract, double* out, int64_t ldo,
                              double alpha, const ItemA* items, int n_items, cudaStream_t stream);

bool contract_kp_supported(int kp);

// W[row][f] = sum_c A[row][c] M[c][f] (items: o_off = row * lda, rows <= 256, pad = subject)
cudaError_t launch_apply_rows(int kp, int a_dtype, const void* A, int64_t lda, const double* M, int64_t mstride,
                              double* W, int K, const ItemA* items, int n_items, cudaStream_t stream);

// 128 x 128 tiles of X^T X (items: l_off/r_off column offsets, pad = 1 on diagonal tiles)
cudaError_t launch_gram_tiles(int x_dtype, const void* X, int64_t ldx, double* out, int64_t ldo,
                              const ItemE* items, int n_items, cudaStream_t stream);

// tcgen05 3xTF32 streaming kernels for fp32 X-hat (tc_fp32.cu)
int tc_np(int k);
bool tc_supported(int k);
// opaque 128-byte CUtensorMap (cuda.h) so this header stays driver-API free
struct alignas(64) TmaMap {
  unsigned long long opaque[16];
};
cudaError_t make_map_f32(TmaMap* m, const float* base, int64_t inner, int64_t outer, int64_t pitch,
                         int box_inner, int box_outer, bool swizzle128);
cudaError_t launch_tc_apass(int np, const TmaMap& tmX, const TmaMap& tmS, int64_t ncontract, float* A, int64_t lda,
                            float alpha, const ItemA* items, int n_items, cudaStream_t st);
cudaError_t launch_tc_bpass(int np, const TmaMap& tmA, const TmaMap& tmXb, int64_t ldx, double* out, int64_t ldo,
                            int orows, const ItemE* items, int n_items, cudaStream_t st);
constexpr int kTcRows = 256;  // A-pass rows per CTA / B-pass TRs per CTA

// int8-sliced fp64 Gram (ozaki.cu): one upper 128 x 128 tile of G_subj
struct OzItem {
  int32_t subj;  // local subject
  int32_t m0;    // first row (TR) of the tile
  int32_t n0;    // first column (TR) of the tile
  int32_t nvb;   // 32-voxel blocks of the subject (of the chunk, k_oz_gram)
  int32_t vb0;   // k_oz_gram: first 32-voxel block (a V chunk of the subject)
  int32_t slot;  // k_oz_gram: output matrix index (the subject, or a V chunk's partial)
};
// where k_oz_gram writes: matrix slot s at g + s gsub, entry (a, b) at
// [a ldg + b] for a, b < nout; column exponents expo[subj ldexp + t], t < nexp
// (entries beyond nexp: the zero columns of a padded record tensor)
struct OzGramOut {
  double* g;
  int64_t ldg, gsub, nout;
  const int32_t* expo;
  int64_t ldexp, nexp;
  // columns the MMAs must cover (T): a tile's N is trimmed to the 16-column
  // multiple that reaches it, and its columns beyond are written as the zeros
  // they are (0 = all of nout)
  int64_t nmma = 0;
};
constexpr int kOzChunkBlocks = 2048;  // 65536 voxels per exact int32 accumulation
constexpr int64_t kOzRecord = 256;    // bytes per (row, 32-column block): 8 slots x 32
// record bytes of the X-hat slices: 8 slots (256 B) for fp64's seven slices,
// 4 slots (128 B) for fp32's four
inline __host__ __device__ int oz_record_bytes(int nsl) { return nsl <= 4 ? 128 : 256; }
cudaError_t make_map_q(TmaMap* m, const int8_t* base, int64_t lq, int64_t rows, int64_t n, int box_rows);
cudaError_t make_map_q5(TmaMap* m, const int8_t* base, int64_t lq, int64_t ldx, int64_t n, int nsl);
// box {32 B, 64 rows, `slots` 32-byte slots of a record, 1}: the leading slots of each record
cudaError_t make_map_q8(TmaMap* m, const int8_t* base, int64_t lq, int64_t rows, int64_t n, int slots = 8);
// int8 slices of the rows of a row-major fp64 matrix (ozaki.cu): 2^e[r] >= max|M[r][:]|
// tile_rows > 0: the tiled layout of the G_i slices (rows per G_i; oz_tiled_bytes per G_i)
// tile_rows < 0: the tiled layout of R'^T for the final W (-tile_rows = kp rows per
// subject): [subject][32-column block][64-row half][8 slots][64 rows][32 B] in the
// SWIZZLE_32B chunk order, kOzRTile bytes per (block, half); rows past kp stay as zeroed
constexpr int64_t kOzRTile = 8 * 64 * 32;
inline int64_t oz_rtiled_bytes(int64_t kp, int64_t ncols) { return (kp + 63) / 64 * (ncols / 32) * kOzRTile; }
cudaError_t launch_oz_slice_rows(const double* M, int64_t ldm, int64_t rows, int64_t ncols, int8_t* q, int64_t lq,
                                 int32_t* expo, cudaStream_t st, int64_t tile_rows = 0);
size_t oz_tiled_bytes(int64_t rows, int64_t ncols);
// B_i = S G_i / 2 into bred[i][f][t] from the row slices of G_i and S (kp <= 128),
// local subjects [first, first + count)
cudaError_t launch_oz_sg(const TmaMap& tmg, const TmaMap& tms, const int32_t* gexp, const int32_t* sexp,
                         double* bred, int64_t ldx, int64_t kp, int64_t ldo, int first, int count, cudaStream_t st);
// the same B_i, stream-K over at most max_ctas persistent CTAs; part holds
// max_ctas x oz_sk_park_bytes(), flag max_ctas int32 (zero between launches)
size_t oz_sk_park_bytes();
cudaError_t launch_oz_sg_sk(const TmaMap& tmg, const TmaMap& tms, const int32_t* gexp, const int32_t* sexp,
                            double* bred, int32_t* part, int32_t* flag, int64_t ldx, int64_t kp, int64_t ldo,
                            int first, int count, int max_ctas, cudaStream_t st);
// R'^T[i] = 2^{e_t} (M_i^T S) / 2 (kp x ldx per subject) for the final int8 W = Xhat R
cudaError_t launch_oz_rt(const double* mmat, const double* S, const int32_t* expo, double* rt, int64_t ldx,
                         int64_t kp, int64_t K, int n_local, cudaStream_t st);
// W rows = Qt (voxel-major X-hat slices) x the row slices of R'^T (kp <= 64)
// (rt: the tiled slices of R'^T, launch_oz_slice_rows with tile_rows = -kp)
cudaError_t launch_oz_w(const TmaMap& tmqt, const TmaMap& tmr, const int8_t* rt, const int32_t* rexp, double* W,
                        const OzItem* items, int n_items, int64_t ldx, int64_t kp, int64_t K, int nsl, cudaStream_t st);
// fp32 X-hat: the same W with the A operand sliced in the kernel from X-hat
// (tmx: fp32 [rows_total][ldx], box {32, 128}, SWIZZLE_128B; xexp: the column
// exponents k_oz_split_f32 used), bit-identical to launch_oz_w's
cudaError_t launch_oz_wx(const TmaMap& tmx, const TmaMap& tmr, const int8_t* rt, const int32_t* xexp,
                         const int32_t* rexp, double* W, const OzItem* items, int n_items, int64_t ldx, int64_t kp,
                         int64_t K, cudaStream_t st);
size_t oz_gram_smem_bytes();
// init E-step on the int8 tensor cores: B_i = G_i^T Xhat_i (G = the N(0,1) draw
// in AMAT) into bred, from G's seven-slice records [i][k][vb] (qg, pitch lqg)
// and Xhat's nslb-slice records; items = one per (subject, 128-TR tile)
cudaError_t launch_oz_tn(const TmaMap& tma, const TmaMap& tmb, const int32_t* aexp, const int32_t* bexp, double* bred,
                         int64_t ldx, int64_t kp, int64_t ldo, int64_t K, const OzItem* items, int n_items, int nslb,
                         cudaStream_t st);
// the same tiles on CTA pairs (tcgen05 cta_group::2, M = 256): items are
// (subject, m0 = first of two row blocks, n0, nvb); tmqb: the records with a
// 64-row box (each CTA stages half of the B rows)
cudaError_t launch_oz_gram2(const TmaMap& tmq, const TmaMap& tmqb, const OzGramOut& o, const OzItem* items,
                            int n_items, int nsl, cudaStream_t st);
// the same for kp <= 64, transposed (M = 128 TRs x N = two slots of 64 features, one
// pass): tmg8 = the draw's records through make_map_q8 (slot-major boxes of 64 rows;
// eight slots, or the first four for four-slice X-hat)
cudaError_t launch_oz_nt(const TmaMap& tmx, const TmaMap& tmg8, const int32_t* aexp, const int32_t* bexp,
                         double* bred, int64_t ldx, int64_t kp, int64_t ldo, int64_t K, const OzItem* items, int n_items,
                         int nslx, cudaStream_t st);
// X_i^T X_i tiles from the nsl-slice records (nsl = 7 for fp64 X-hat, 4 for
// fp32); also G_i^T G_i of the init draw from its seven-slice records
cudaError_t launch_oz_gram(const TmaMap& tmq, const OzGramOut& o, const OzItem* items, int n_items, int nsl,
                           cudaStream_t st);

// accurate polar transform (qr_polar.cu): Householder TSQR of a tall V x K
// matrix, then a one-sided Jacobi SVD of R -> M = V diag(1/sigma) V^T
struct QrJob {
  const double* a;  // first row of this job's matrix (or the stacked factors of the last level)
  int64_t lda;
  int64_t rows;
  int64_t rpc;      // rows per CTA
  double* rout;     // nctas x (K x K) upper-triangular factors
  int32_t nctas;
  int32_t pad;
};
struct SvdJob {
  const double* r;  // K x K factor (pitch K)
  double* m;        // output transform, pitch ldm, zero-padded to mp x mp
  int64_t ldm;
  int32_t mp;
  int32_t subject;  // reported with RankError
  double* vg;       // K x K global scratch for V when svd_needs_global_v(K), else null
};
struct TsqrSchedule {
  struct Job {
    int64_t rows, rpc;
    int nctas;
    int64_t out_off;  // doubles into this level's output buffer
  };
  std::vector<std::vector<Job>> levels;  // level 0 reads the matrices, level L the factors of L - 1
  int64_t buf_doubles = 0;               // per ping-pong buffer
};
bool qr_polar_supported(int K);
bool svd_needs_global_v(int K);
int tsqr_block_rows(int K);
TsqrSchedule tsqr_schedule(const std::vector<int64_t>& rows, int K, int target_ctas);
std::vector<std::vector<QrJob>> tsqr_jobs(const TsqrSchedule& s, const std::vector<const double*>& a,
                                          const std::vector<int64_t>& lda, int K, double* buf0, double* buf1,
                                          std::vector<const double*>* r_final);
int tsqr_max_ctas(const std::vector<TsqrSchedule::Job>& lvl);
cudaError_t launch_tsqr(const QrJob* jobs_dev, int n_jobs, int max_ctas, int K, cudaStream_t st);
cudaError_t launch_svd_polar(const SvdJob* jobs_dev, int n_jobs, int K, int32_t* status, const int32_t* iter,
                             cudaStream_t st);

// transforms (transform.cu): xp[r][c] = x[r][c] - mu[r] (fp64, zero pad to ldp),
// and out = A B + bias 1^T (A: V x K, B: K x N, K <= 128)
cudaError_t launch_center_stage(const void* x, int x_dtype, int64_t ldx, const double* mu, int64_t v, int64_t t,
                                double* xp, int64_t ldp, cudaStream_t st);
bool gemm_nn_bias_supported(int K);
cudaError_t launch_gemm_nn_bias(const double* A, int64_t lda, const double* B, int64_t ldb, const double* bias,
                                double* out, int64_t ldo, int64_t V, int K, int64_t N, cudaStream_t st);

// thread-local message returned by srm_last_error() (defined in capi.cu)
void set_last_error(const char* where, cudaError_t e);

}  // namespace srm

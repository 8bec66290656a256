// C ABI of libsrm_b200.so (declared in include/srm_b200.h).
//
// A plan is the device-side state of one worker's share of an SRM fit
// (srm.py:216-327): the concatenated X-hat of its subjects, the per-subject
// E-step term table, the K x K state and the static work decomposition of the
// streaming kernels.  The caller (the Python host layer) allocates one device
// workspace; the plan carves it into regions, uploads its work tables once in
// srm_plan_bind, and every phase function below only enqueues kernels on the
// given stream -- no host synchronisation, so a whole iteration can be
// captured into a CUDA graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/srm_b200.h"
#include "kernels.h"
#include "plan.h"

using namespace srm;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SRM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

enum Internal {
  I_ROWSQ = SRM_R_COUNT,
  I_CMAT,
  I_TAILSCR,
  I_SINV,
  I_SSPART,
  I_TAILPART,
  I_PART,
  I_BRED,
  I_QMAT,
  I_QSCR,
  I_CROSSP,
  I_SUBJ,
  I_ORDER,
  I_ORDER_LOCAL,
  I_ITEMS_EX,
  I_ITEMS_EA,
  I_ITEMS_A,
  I_ST,
  I_ITEMS_GRAM,
  I_ITEMS_BG,
  I_AF,
  I_SF,
  I_ITEMS_TB,
  I_ITEMS_TA,
  I_ITEMS_TG,
  I_OZQ,
  I_OZCMAX,
  I_OZEXP,
  I_ITEMS_OZ,
  I_GFBPART,
  I_GFBCOUNT,
  I_OZG,
  I_OZGEXP,
  I_OZS,
  I_OZSEXP,
  I_OZR,
  I_OZREXP,
  I_ITEMS_OW,
  I_OZSKPART,
  I_OZSKFLAG,
  I_QRBUF0,
  I_QRBUF1,
  I_QRJOBS,
  I_SVDJOBS,
  I_NSG,
  I_OZGIEXP,
  I_OZGICMAX,
  I_ITEMS_TN,
  I_ITEMS_GG,
  I_ITEMS_OZ2,
  I_XCOUNTS,
  I_COUNT
};

}  // namespace

void srm::set_last_error(const char* where, cudaError_t e) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
}

// side streams + fork/join events of a plan (the stage lists' lanes 1 and 2)
struct Lanes {
  cudaStream_t side[3];
  cudaEvent_t fork[3], join[3];
};

struct srm_plan {
  int dtype = SRM_F64;
  int n_local = 0;
  std::vector<int64_t> V;
  int64_t T = 0, K = 0, ldx = 0, kp = 0, ldo = 0;
  int iterations = 0;
  int world = 1, rank = 0;
  std::vector<int32_t> counts;
  int flags = 0;
  int n_total = 0, max_local = 0, global0 = 0;
  int n_slots = 0, slot0 = 0;
  int64_t rows_total = 0;
  std::vector<int64_t> row_off;
  int64_t chunk_rows = 0;
  std::vector<int64_t> chunk0, nchunk;
  int64_t chunks_total = 0;
  std::vector<ItemE> items_ex, items_ea, items_gram, items_bg, items_tb, items_tg;
  int np = 0;  // tensor-core feature padding
  std::vector<ItemA> items_a, items_ta;
  std::vector<int64_t> subj;
  std::vector<int32_t> order, order_local;
  int64_t off[I_COUNT] = {0};
  int64_t size[I_COUNT] = {0};
  int64_t total_bytes = 0;
  char* ws = nullptr;
  DevPlan dp{};
  cudaStream_t cap_stream = nullptr;
  Lanes lanes{};            // side lanes of the stage lists (created on first use)
  bool lanes_ready = false;
  std::vector<cudaEvent_t> gram_events;  // per-batch "slices ready" of the pipelined Gram
  cudaStream_t hi_stream = nullptr;      // high-priority stream of the pipelined Gram
  cudaStream_t hi_stream2 = nullptr;     // ... and of its CTA-pair tiles
  std::vector<cudaEvent_t> pair_events;  // per-batch "pair tiles done"
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  TmaMap tm_x_a, tm_s, tm_a, tm_x_b;  // tensor-core path TMA maps (bound at srm_plan_bind)
  std::vector<OzItem> items_oz;       // int8-sliced Gram tiles (SRM_FLAG_GRAM_I8) on single CTAs
  std::vector<OzItem> items_oz2;      // with gram_pairs: (subject, 256-row pair, n0) tiles on CTA pairs
  bool gram_pairs = false;            // off-diagonal tile pairs on CTA pairs (k_oz_gram2)
  // one rank, polar_cross: the next E-step's K x K tail (k_tail_kk, needs only
  // Sigma_s^{-1} and rho0) runs at the end of the M-step beside apply_m
  bool early_kk = false;
  TmaMap tm_qb;                       // the X-hat records with a 64-row box (the pairs' B halves)
  int64_t oz_lq = 0, max_v = 0;       // bytes per sliced TR row; largest local V
  int oz_nsl = 7;                     // int8 slices per X-hat value: 7 (fp64), 4 (fp32)
  TmaMap tm_q;
  bool oz_sg = false;                 // per-iteration B = S G / 2 from int8 row slices (kp <= 64)
  int64_t oz_lqg = 0;                 // bytes per sliced row of G_i / S / R'^T / Qt
  TmaMap tm_g, tm_sq;
  bool oz_w = false;                  // final W = Xhat R from the int8 slices (needs oz_sg)
  std::vector<OzItem> items_ow;       // 128-voxel tiles of the final int8 W = Xhat R
  std::vector<OzItem> items_tn;       // (subject, 128-TR tile) of the int8 init term B_0 = G^T Xhat
  std::vector<OzItem> items_gg;       // (subject, V chunk) of the int8 G^T G of the init draw (kp > 64)
  int64_t oz_lqg_init = 0;            // bytes per sliced row (feature) of the init draw G (records in WOUT)
  TmaMap tm_gi, tm_gi64;
  std::vector<cudaEvent_t> post_events;  // batched int8 Gram: batch b's Gram done (mirror / G slices follow on hi_stream2)
  std::vector<char> sliced;           // srm_prepare_gram_range has been enqueued for the subject
  std::vector<int> ow_first;          // [n_local + 1]: first items_ow entry of each subject
  TmaMap tm_q32, tm_r;
  TmaMap tm_xw;     // fp32 X-hat, box {32 TRs, 128 voxels}, SWIZZLE_128B (the final W's in-kernel slicing)
  bool ozw_x = false;  // fp32 X-hat: oz_w slices X-hat in the kernel (opt-in, SRM_B200_OZW=x)
  bool sk_off = false;                // SRM_B200_SG_PER_TILE=1: per-tile B = S G / 2 (test knob)
  int sk_ctas = 0;                    // stream-K B = S G / 2: persistent CTAs (SMs less two for the side lane)
  TsqrSchedule qr;                    // SRM_FLAG_EXACT_POLAR: TSQR levels over the local A_i (job table: level-major)
};

namespace {

int64_t esize(int dtype) { return dtype == SRM_F64 ? 8 : 4; }

void layout(srm_plan* p) {
  const int64_t kp2 = p->kp * p->kp;
  const int ntile_tail = (int)((p->ldx + 31) / 32);
  const int ntile_apply = (int)((p->ldx + apply_cols_for(p->kp) - 1) / apply_cols_for(p->kp));
  const int64_t term_stride = p->kp * p->ldx + kRecScalars;
  const int64_t red_stride = p->kp * p->ldx + kRedScalars;
  const int64_t hist_stride = SRM_H_RHO2 + std::max(p->n_local, 1);
  int64_t sz[I_COUNT] = {0};
  sz[SRM_R_XHAT] = p->rows_total * p->ldx * esize(p->dtype);
  sz[SRM_R_AMAT] = p->rows_total * p->kp * 8;
  // W_i (final) -- and, on int8 Gram plans, the slices of the init draw G before it
  sz[SRM_R_WOUT] = std::max(p->rows_total * p->K * 8, (int64_t)p->n_local * p->K * p->oz_lqg_init);
  sz[SRM_R_MU] = p->rows_total * 8;
  sz[SRM_R_TERMS] = (int64_t)p->n_slots * term_stride * 8;
  sz[SRM_R_RED] = red_stride * 8;
  sz[SRM_R_REDLOCAL] = red_stride * 8;
  sz[SRM_R_S] = p->kp * p->ldx * 8;
  sz[SRM_R_SIGMA] = kp2 * 8;
  sz[SRM_R_HIST] = (int64_t)std::max(p->iterations, 1) * hist_stride * 8;
  sz[SRM_R_STATUS] = 32;  // status word + iteration counter
  sz[SRM_R_MMAT] = (int64_t)p->n_local * kp2 * 8;
  sz[SRM_R_SCAL] = (int64_t)p->n_local * 8 * 8;
  sz[SRM_R_GRAM] = (p->flags & SRM_FLAG_GRAM) ? (int64_t)p->n_local * p->ldx * p->ldx * 8 : 0;
  sz[SRM_R_VAR] = kp2 * 8;
  // SRM_FLAG_COLBLOCK exchange buffers
  const bool cb = (p->flags & SRM_FLAG_COLBLOCK) != 0;
  const int64_t xw = (p->ldx + p->world - 1) / p->world;
  const int64_t xrec = p->kp * xw + kRecScalars, xred = p->kp * xw + kRedScalars;
  sz[SRM_R_XSEND] = cb ? (int64_t)p->world * p->max_local * xrec * 8 : 0;
  sz[SRM_R_XRECV] = sz[SRM_R_XSEND];
  sz[SRM_R_XRED] = cb ? (int64_t)p->world * xred * 8 : 0;
  sz[I_XCOUNTS] = cb ? (int64_t)p->world * 4 : 0;
  sz[I_ROWSQ] = p->rows_total * 8;
  sz[I_CMAT] = kp2 * 8;
  sz[I_TAILSCR] = kTailScalars * 8;
  sz[I_SINV] = kp2 * 8;
  sz[I_SSPART] = (int64_t)ntile_tail * kp2 * 8;
  sz[I_TAILPART] = (int64_t)ntile_tail * 4 * 8;
  sz[I_PART] = p->chunks_total * p->kp * p->ldo * 8;
  sz[I_BRED] = (int64_t)p->n_local * p->kp * p->ldo * 8;
  sz[I_QMAT] = (int64_t)p->n_local * kp2 * 8;
  sz[I_QSCR] = (int64_t)p->n_local * kp2 * 8;
  sz[I_CROSSP] = (int64_t)p->n_local * ntile_apply * 8;
  sz[I_SUBJ] = (int64_t)p->subj.size() * 8;
  sz[I_ORDER] = (int64_t)p->order.size() * 4;
  sz[I_ORDER_LOCAL] = (int64_t)p->order_local.size() * 4;
  sz[I_ITEMS_EX] = (int64_t)p->items_ex.size() * sizeof(ItemE);
  sz[I_ITEMS_EA] = (int64_t)p->items_ea.size() * sizeof(ItemE);
  sz[I_ITEMS_A] = (int64_t)p->items_a.size() * sizeof(ItemA);
  sz[I_ST] = p->ldx * p->kp * 8;
  sz[I_ITEMS_GRAM] = (int64_t)p->items_gram.size() * sizeof(ItemE);
  sz[I_ITEMS_BG] = (int64_t)p->items_bg.size() * sizeof(ItemE);
  const bool tc = (p->flags & SRM_FLAG_TC) != 0;
  sz[I_AF] = tc ? p->rows_total * p->np * 4 : 0;
  sz[I_SF] = tc ? 2 * (int64_t)p->np * p->ldx * 4 : 0;
  sz[I_ITEMS_TB] = (int64_t)p->items_tb.size() * sizeof(ItemE);
  sz[I_ITEMS_TA] = (int64_t)p->items_ta.size() * sizeof(ItemA);
  sz[I_ITEMS_TG] = (int64_t)p->items_tg.size() * sizeof(ItemE);
  const bool i8 = (p->flags & SRM_FLAG_GRAM_I8) != 0;
  sz[I_OZQ] = i8 ? (int64_t)p->n_local * p->ldx * p->oz_lq : 0;
  sz[I_OZCMAX] = i8 ? (int64_t)p->n_local * p->ldx * 8 : 0;
  sz[I_OZEXP] = i8 ? (int64_t)p->n_local * p->ldx * 4 : 0;
  sz[I_ITEMS_OZ] = (int64_t)p->items_oz.size() * sizeof(OzItem);
  sz[I_ITEMS_OZ2] = (int64_t)p->items_oz2.size() * sizeof(OzItem);
  const int gfb_chunks = (int)((p->ldx + kGfbCols - 1) / kGfbCols);
  sz[I_GFBPART] = (int64_t)p->n_local * gfb_chunks * kp2 * 8;
  sz[I_GFBCOUNT] = (int64_t)p->n_local * 4;
  sz[I_OZG] = p->oz_sg ? (int64_t)p->n_local * (int64_t)oz_tiled_bytes(p->ldx, p->ldx) : 0;
  sz[I_OZGEXP] = p->oz_sg ? (int64_t)p->n_local * p->ldx * 4 : 0;
  sz[I_OZS] = p->oz_sg ? p->kp * p->oz_lqg : 0;
  sz[I_OZSEXP] = p->oz_sg ? p->kp * 4 : 0;
  sz[I_OZR] = p->oz_w ? (int64_t)p->n_local * oz_rtiled_bytes(p->kp, p->ldx) : 0;  // zeroed at bind: rows past kp
  sz[I_OZREXP] = p->oz_w ? (int64_t)p->n_local * p->kp * 4 : 0;
  sz[I_ITEMS_OW] = (int64_t)p->items_ow.size() * sizeof(OzItem);
  sz[I_OZSKPART] = p->oz_sg ? (int64_t)p->sk_ctas * oz_sk_park_bytes() : 0;
  sz[I_OZSKFLAG] = p->oz_sg ? (int64_t)p->sk_ctas * 4 : 0;
  const bool exact = (p->flags & SRM_FLAG_EXACT_POLAR) != 0;
  sz[I_QRBUF0] = exact ? p->qr.buf_doubles * 8 : 0;
  sz[I_QRBUF1] = exact ? p->qr.buf_doubles * 8 : 0;
  sz[I_QRJOBS] = exact ? (int64_t)p->qr.levels.size() * p->n_local * (int64_t)sizeof(QrJob) : 0;
  sz[I_SVDJOBS] = exact ? (int64_t)p->n_local * (int64_t)sizeof(SvdJob) : 0;
  sz[I_NSG] = ns_polar_g_supported((int)p->kp) ? (int64_t)p->n_local * 4 * kp2 * 8 : 0;
  sz[I_OZGIEXP] = p->oz_lqg_init ? (int64_t)p->n_local * p->K * 4 : 0;
  sz[I_OZGICMAX] = p->oz_lqg_init ? (int64_t)p->n_local * p->K * 8 : 0;
  sz[I_ITEMS_TN] = (int64_t)p->items_tn.size() * sizeof(OzItem);
  sz[I_ITEMS_GG] = (int64_t)p->items_gg.size() * sizeof(OzItem);
  int64_t cur = 0;
  for (int r = 0; r < I_COUNT; ++r) {
    p->off[r] = cur;
    p->size[r] = sz[r];
    cur += round_up(sz[r], 256);
  }
  p->total_bytes = std::max<int64_t>(cur, 256);
  DevPlan& d = p->dp;
  d.n_local = p->n_local;
  d.sub0 = 0;
  d.nsub = p->n_local;
  d.n_total = p->n_total;
  d.n_order = (int)p->order.size();
  d.flags = p->flags;
  d.xf32 = p->dtype == SRM_F32 ? 1 : 0;
  // the M-step polar is one of the Newton-Schulz kernels (launch_eig_polar's
  // dispatch), which then also form the cross term; not on the exact route
  d.polar_cross = !(p->flags & SRM_FLAG_EXACT_POLAR) &&
                  (ns_polar_supported((int)p->kp) || ns_polar_g_supported((int)p->kp)) &&
                  !getenv("SRM_B200_APPLY_CROSS");
  p->early_kk = d.polar_cross && p->world == 1;
  d.T = p->T;
  d.K = p->K;
  d.ldx = p->ldx;
  d.kp = p->kp;
  d.ldo = p->ldo;
  d.ntile_apply = ntile_apply;
  d.apply_cols = apply_cols_for(p->kp);
  d.ntile_tail = ntile_tail;
  d.gfb_chunks = gfb_chunks;
  d.term_stride = term_stride;
  d.red_stride = red_stride;
  d.hist_stride = hist_stride;
}

template <typename T>
T* region(srm_plan* p, int r) {
  return reinterpret_cast<T*>(p->ws + p->off[r]);
}

void build_work(srm_plan* p) {
  // V-chunking of the split-V contraction: about 8 waves of 2 CTAs per SM
  const int64_t ntiles = (p->ldx + 127) / 128;
  const int64_t target_items = 148 * 2 * 8;
  int64_t cr = round_up(std::max<int64_t>(1, p->rows_total * ntiles / target_items), 16);
  cr = std::max<int64_t>(cr, 256);
  p->chunk_rows = cr;
  p->chunk0.assign(p->n_local, 0);
  p->nchunk.assign(p->n_local, 0);
  int64_t c = 0;
  for (int i = 0; i < p->n_local; ++i) {
    p->chunk0[i] = c;
    p->nchunk[i] = std::max<int64_t>(1, (p->V[i] + cr - 1) / cr);
    c += p->nchunk[i];
  }
  p->chunks_total = c;
  p->items_ex.clear();
  p->items_ea.clear();
  p->items_a.clear();
  for (int i = 0; i < p->n_local; ++i) {
    for (int64_t ch = 0; ch < p->nchunk[i]; ++ch) {
      const int64_t r0 = p->row_off[i] + ch * cr;
      const int64_t rows = std::max<int64_t>(0, std::min<int64_t>(cr, p->V[i] - ch * cr));
      const int64_t obase = (p->chunk0[i] + ch) * p->kp * p->ldo;
      for (int64_t n0 = 0; n0 < p->ldx; n0 += 128) {
        ItemE it;
        it.l_off = r0 * p->kp;
        it.r_off = r0 * p->ldx + n0;
        it.o_off = obase + n0;
        it.rows = (int32_t)rows;
        it.ncols = (int32_t)std::min<int64_t>(128, p->ldx - n0);
        it.mrows = (int32_t)p->kp;
        it.pad = 0;
        p->items_ex.push_back(it);
      }
      ItemE ia;
      ia.l_off = r0 * p->kp;
      ia.r_off = r0 * p->kp;
      ia.o_off = obase + p->ldx;
      ia.rows = (int32_t)rows;
      ia.ncols = (int32_t)p->kp;
      ia.mrows = (int32_t)p->kp;
      ia.pad = 0;
      p->items_ea.push_back(ia);
    }
    for (int64_t r = 0; r < p->V[i]; r += 128) {
      ItemA it;
      it.x_off = (p->row_off[i] + r) * p->ldx;
      it.o_off = (p->row_off[i] + r) * p->kp;
      it.rows = (int32_t)std::min<int64_t>(128, p->V[i] - r);
      it.pad = i;
      p->items_a.push_back(it);
    }
  }
  // Gram path: one-time X_i^T X_i (upper 128 x 128 tiles) and per-iteration B_i = S G_i / 2
  p->items_gram.clear();
  p->items_bg.clear();
  if (p->flags & SRM_FLAG_GRAM) {
    for (int i = 0; i < p->n_local; ++i) {
      for (int64_t m0 = 0; m0 < p->ldx; m0 += 128) {
        for (int64_t n0 = m0; n0 < p->ldx; n0 += 128) {
          ItemE it;
          it.l_off = p->row_off[i] * p->ldx + m0;
          it.r_off = p->row_off[i] * p->ldx + n0;
          it.o_off = (int64_t)i * p->ldx * p->ldx + m0 * p->ldx + n0;
          it.rows = (int32_t)p->V[i];
          it.ncols = (int32_t)std::min<int64_t>(128, p->ldx - n0);
          it.mrows = (int32_t)std::min<int64_t>(128, p->ldx - m0);
          it.pad = (m0 == n0) ? 1 : 0;
          p->items_gram.push_back(it);
        }
      }
      for (int64_t n0 = 0; n0 < p->ldx; n0 += 128) {
        ItemE it;
        it.l_off = 0;
        it.r_off = (int64_t)i * p->ldx * p->ldx + n0;
        it.o_off = (int64_t)i * p->kp * p->ldo + n0;
        it.rows = (int32_t)p->ldx;
        it.ncols = (int32_t)std::min<int64_t>(128, p->ldx - n0);
        it.mrows = (int32_t)p->kp;
        it.pad = 0;
        p->items_bg.push_back(it);
      }
    }
  }
  // int8-sliced Gram: the same upper tiles, slices [n_local][ldx][oz_lq]
  p->items_oz.clear();
  p->items_oz2.clear();
  p->max_v = 0;
  for (int i = 0; i < p->n_local; ++i) p->max_v = std::max(p->max_v, p->V[i]);
  p->oz_nsl = p->dtype == SRM_F64 ? 7 : 4;
  p->oz_lq = round_up(std::max<int64_t>(p->max_v, 1), 32) / 32 * oz_record_bytes(p->oz_nsl);
  p->oz_sg = (p->flags & SRM_FLAG_GRAM_I8) && p->kp <= 128;
  p->oz_lqg = p->ldx / 32 * kOzRecord;
  p->oz_w = p->oz_sg;
  {
    // opt-in (SRM_B200_OZW=x): bit-identical, but measured 3-4x slower than the
    // records path so far (cfg 5: 139 vs 37 ms)
    const char* env = getenv("SRM_B200_OZW");
    p->ozw_x = p->oz_w && p->dtype == SRM_F32 && env && !strcmp(env, "x");
  }
  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        sms <= 0) {
      cudaGetLastError();
      sms = 148;
    }
    p->sk_ctas = std::max(1, sms - 2);
    // test knob: the per-tile grid (k_oz_rowgemm<kRowSG>) instead of stream-K, to show both agree bit for bit
    const char* env = getenv("SRM_B200_SG_PER_TILE");
    p->sk_off = env && env[0] == '1';
  }
  p->items_ow.clear();
  p->ow_first.assign(1, 0);
  for (int i = 0; i < p->n_local; ++i) {
    if (p->oz_w)
      for (int64_t v0 = 0; v0 < p->V[i]; v0 += 128)
        p->items_ow.push_back({i, (int32_t)v0, (int32_t)(p->row_off[i] + v0),
                               (int32_t)std::min<int64_t>(128, p->V[i] - v0)});
    p->ow_first.push_back((int)p->items_ow.size());
  }
  {
    // SRM_B200_GRAM_PAIRS=1: the off-diagonal tiles of each column block two
    // row blocks at a time on CTA pairs (k_oz_gram2, cta_group::2, M = 256:
    // each CTA stages half of the shared B rows, a quarter less operand
    // traffic through the tensor core's shared-memory port), the diagonal
    // tiles and the odd leftover on single CTAs -- the same 36 tiles at T =
    // 1000, none below the diagonal.  Bit-identical to the single-CTA grid.
    // Opt-in: the pair and single tiles run concurrently in each batch of the
    // pipelined Gram, and the Gram stage alone is 10% faster on four-slice
    // records (cfg 5: 61 vs 69 ms), but the whole fit is not (166 vs 164 ms at
    // the power-capped clock); on seven-slice records the pairs are slower
    const char* env = getenv("SRM_B200_GRAM_PAIRS");
    p->gram_pairs = env && env[0] == '1';
  }
  if (p->flags & SRM_FLAG_GRAM_I8) {
    for (int i = 0; i < p->n_local; ++i) {
      const OzItem base{i, 0, 0, (int32_t)((p->V[i] + 31) / 32), 0, i};
      for (int64_t n0 = 0; n0 < p->ldx; n0 += 128) {
        int64_t m0 = 0;
        if (p->gram_pairs)
          for (; m0 + 128 < n0; m0 += 256) {
            OzItem it = base;
            it.m0 = (int32_t)m0;
            it.n0 = (int32_t)n0;
            p->items_oz2.push_back(it);
          }
        for (; m0 <= n0; m0 += 128) {
          OzItem it = base;
          it.m0 = (int32_t)m0;
          it.n0 = (int32_t)n0;
          p->items_oz.push_back(it);
        }
      }
    }
  }
  // the init E-step term B_0 = G^T Xhat from int8 slices too (with the int8 B = S G)
  p->items_tn.clear();
  p->items_gg.clear();
  p->oz_lqg_init = 0;
  if (p->oz_sg) {
    p->oz_lqg_init = round_up(std::max<int64_t>(p->max_v, 1), 32) / 32 * 256;
    for (int i = 0; i < p->n_local; ++i)
      for (int64_t n0 = 0; n0 < p->ldx; n0 += 128)
        p->items_tn.push_back({i, 0, (int32_t)n0, (int32_t)((p->V[i] + 31) / 32)});
    // kp > 64: G^T G of the draw from its slices too, one partial per split-V
    // chunk (the chunk count of the DMMA contraction it replaces, 32-voxel
    // aligned), summed by reduce_chunks in the same order
    if (p->kp > 64)
      for (int i = 0; i < p->n_local; ++i) {
        const int64_t nb = (p->V[i] + 31) / 32, nc = p->nchunk[i];
        for (int64_t ch = 0; ch < nc; ++ch) {
          const int64_t b0 = ch * nb / nc, b1 = (ch + 1) * nb / nc;
          p->items_gg.push_back({i, 0, 0, (int32_t)(b1 - b0), (int32_t)b0, (int32_t)(p->chunk0[i] + ch)});
        }
      }
  }
  // tensor-core path: A-pass row tiles (A in the fp32 [rows][np] region) and
  // B-pass tiles of 128 TRs over the same V chunks
  p->items_tb.clear();
  p->items_ta.clear();
  p->items_tg.clear();
  if (p->flags & SRM_FLAG_TC) {
    // exact fp64 A^T A of the stored fp32 A (final W only): same V chunks
    for (int i = 0; i < p->n_local; ++i) {
      for (int64_t ch = 0; ch < p->nchunk[i]; ++ch) {
        const int64_t r0 = p->row_off[i] + ch * cr;
        ItemE g;
        g.l_off = r0 * p->np;
        g.r_off = r0 * p->np;
        g.o_off = (p->chunk0[i] + ch) * p->kp * p->ldo + p->ldx;
        g.rows = (int32_t)std::max<int64_t>(0, std::min<int64_t>(cr, p->V[i] - ch * cr));
        g.ncols = (int32_t)p->kp;
        g.mrows = (int32_t)p->kp;
        g.pad = 0;
        p->items_tg.push_back(g);
      }
    }
    for (int i = 0; i < p->n_local; ++i) {
      for (int64_t r = 0; r < p->V[i]; r += kTcRows) {
        ItemA t;
        t.x_off = (p->row_off[i] + r) * p->ldx;
        t.o_off = (p->row_off[i] + r) * p->np;
        t.rows = (int32_t)std::min<int64_t>(kTcRows, p->V[i] - r);
        t.pad = i;
        p->items_ta.push_back(t);
      }
    }
    for (int i = 0; i < p->n_local; ++i) {
      for (int64_t ch = 0; ch < p->nchunk[i]; ++ch) {
        const int64_t r0 = p->row_off[i] + ch * cr;
        const int64_t rows = std::max<int64_t>(0, std::min<int64_t>(cr, p->V[i] - ch * cr));
        const int64_t obase = (p->chunk0[i] + ch) * p->kp * p->ldo;
        for (int64_t n0 = 0; n0 < p->ldx; n0 += kTcRows) {
          ItemE it;
          it.l_off = r0 * p->np;
          it.r_off = r0 * p->ldx + n0;
          it.o_off = obase + n0;
          it.rows = (int32_t)rows;
          it.ncols = (int32_t)std::min<int64_t>(kTcRows, p->ldx - n0);
          it.mrows = (int32_t)p->kp;
          it.pad = 0;
          p->items_tb.push_back(it);
        }
      }
    }
  }
  // exact polar route: TSQR levels over every local A_i (V_i x K rows of AMAT)
  p->qr = TsqrSchedule();
  if (p->flags & SRM_FLAG_EXACT_POLAR) p->qr = tsqr_schedule(p->V, (int)p->K, 296);
  // subject table
  p->subj.assign((size_t)p->n_local * kSubjCols, 0);
  for (int i = 0; i < p->n_local; ++i) {
    int64_t* s = &p->subj[(size_t)i * kSubjCols];
    s[SC_ROW_OFF] = p->row_off[i];
    s[SC_V] = p->V[i];
    s[SC_CHUNK0] = p->chunk0[i];
    s[SC_NCHUNK] = p->nchunk[i];
    s[SC_GLOBAL] = p->global0 + i;
    s[SC_SLOT] = p->slot0 + i;
  }
  // record order: ascending global subject index
  p->order.clear();
  p->order_local.clear();
  for (int i = 0; i < p->n_local; ++i) p->order_local.push_back(p->slot0 + i);
  if (p->flags & SRM_FLAG_ORDERED) {
    for (int r = 0; r < p->world; ++r)
      for (int j = 0; j < p->counts[r]; ++j) p->order.push_back(r * p->max_local + j);
  } else {
    p->order = p->order_local;
  }
}

void set_pointers(srm_plan* p) {
  DevPlan& d = p->dp;
  d.xhat = p->ws + p->off[SRM_R_XHAT];
  d.amat = region<double>(p, SRM_R_AMAT);
  d.wout = region<double>(p, SRM_R_WOUT);
  d.mu = region<double>(p, SRM_R_MU);
  d.rowsq = region<double>(p, I_ROWSQ);
  d.terms = region<double>(p, SRM_R_TERMS);
  d.red = region<double>(p, SRM_R_RED);
  d.redlocal = region<double>(p, SRM_R_REDLOCAL);
  d.S = region<double>(p, SRM_R_S);
  d.sigma = region<double>(p, SRM_R_SIGMA);
  d.var = region<double>(p, SRM_R_VAR);
  d.cmat = region<double>(p, I_CMAT);
  d.tailscr = region<double>(p, I_TAILSCR);
  d.sinv = region<double>(p, I_SINV);
  d.sspart = region<double>(p, I_SSPART);
  d.tailpart = region<double>(p, I_TAILPART);
  d.part = region<double>(p, I_PART);
  d.bred = region<double>(p, I_BRED);
  d.gfb_part = region<double>(p, I_GFBPART);
  d.cmax = (p->flags & SRM_FLAG_GRAM_I8) ? region<unsigned long long>(p, I_OZCMAX) : nullptr;
  d.gfb_count = region<int32_t>(p, I_GFBCOUNT);
  d.mmat = region<double>(p, SRM_R_MMAT);
  d.qmat = region<double>(p, I_QMAT);
  d.qscr = region<double>(p, I_QSCR);
  d.crossp = region<double>(p, I_CROSSP);
  d.scal = region<double>(p, SRM_R_SCAL);
  d.nsg = p->size[I_NSG] ? region<double>(p, I_NSG) : nullptr;
  d.st = region<double>(p, I_ST);
  d.gram = p->size[SRM_R_GRAM] ? region<double>(p, SRM_R_GRAM) : nullptr;
  d.af = p->size[I_AF] ? region<float>(p, I_AF) : nullptr;
  d.sf = p->size[I_SF] ? region<float>(p, I_SF) : nullptr;
  d.np = p->np;
  d.hist = region<double>(p, SRM_R_HIST);
  d.status = region<int32_t>(p, SRM_R_STATUS);
  d.iter = d.status + 4;
  d.n_hist = std::max(p->iterations, 1);
  d.subj = region<int64_t>(p, I_SUBJ);
  d.order = region<int32_t>(p, I_ORDER);
  d.world = p->world;
  d.rank = p->rank;
  d.max_local = p->max_local;
  d.xw = (int)((p->ldx + p->world - 1) / p->world);
  d.xrec = p->kp * d.xw + kRecScalars;
  d.xred = p->kp * d.xw + kRedScalars;
  const bool cbx = (p->flags & SRM_FLAG_COLBLOCK) != 0;
  d.xsend = cbx ? region<double>(p, SRM_R_XSEND) : nullptr;
  d.xrecv = cbx ? region<double>(p, SRM_R_XRECV) : nullptr;
  d.xredbuf = cbx ? region<double>(p, SRM_R_XRED) : nullptr;
  d.xcounts = cbx ? region<int32_t>(p, I_XCOUNTS) : nullptr;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int check(cudaError_t e, const char* where) { return e == cudaSuccess ? SRM_OK : cuda_fail(e, where); }

struct Stage {
  const char* name;
  std::function<cudaError_t(cudaStream_t)> fn;
  int lane = 0;       // 1 or 2: on that side stream
  bool join = false;  // both side streams' work completes before this stage
  bool fork = true;   // a side-lane stage starts after everything issued on the main lane so far
};

void contraction_stages(srm_plan* p, std::vector<Stage>& out) {
  const DevPlan& d = p->dp;
  out.push_back({"contract_e_xhat", [p, d](cudaStream_t st) {
                   return launch_contract_e((int)p->kp, SRM_F64, p->dtype, d.amat, p->kp, d.xhat, p->ldx, d.part, p->ldo, 1.0,
                                            region<ItemE>(p, I_ITEMS_EX), (int)p->items_ex.size(), st);
                 }});
  out.push_back({"contract_e_gram", [p, d](cudaStream_t st) {
                   return launch_contract_e((int)p->kp, SRM_F64, SRM_F64, d.amat, p->kp, d.amat, p->kp, d.part, p->ldo, 1.0,
                                            region<ItemE>(p, I_ITEMS_EA), (int)p->items_ea.size(), st);
                 }});
  out.push_back({"reduce_chunks", [d](cudaStream_t st) { return launch_reduce_chunks(d, st); }});
}

std::vector<Stage> e_stages(srm_plan* p) {
  const DevPlan& d = p->dp;
  std::vector<Stage> v;
  // var_s and C (needs only Sigma_s^{-1} and rho0) beside the ordered sum --
  // or already done by the previous M-step (early_kk)
  if (!p->early_kk) v.push_back({"tail_kk", [d](cudaStream_t st) { return launch_tail_kk(d, st); }, 1});
  if (p->flags & SRM_FLAG_ORDERED) {
    const int n = (int)p->order.size();
    bool ident = true;
    for (int j = 0; j < n; ++j) ident = ident && p->order[j] == j;
    v.push_back({"reduce_terms", [d, n, ident](cudaStream_t st) {
                   return launch_reduce_terms(d, d.red, d.order, n, st, ident);
                 }});
  }
  v.push_back({"tail_s", [d](cudaStream_t st) { return launch_tail_s(d, st); }, 0, true});
  // Sigma_s, the LL and the next E-step's Sigma_s^{-1} on the side lane: the
  // M-step needs only S (tail_s) until finalize_rho reads tr(Sigma_s)
  v.push_back({"tail_sigma", [d](cudaStream_t st) { return launch_tail_sigma(d, st); }, 1});
  v.push_back({"tail_inv", [d](cudaStream_t st) { return launch_tail_inv(d, st); }, 1});
  return v;
}

// rho_i^2 of the M-step, then the device iteration counter moves on
void push_finalize_rho(const DevPlan& d, std::vector<Stage>& v) {
  // joins the side lane: tr(Sigma_s) comes from tail_sigma
  if (finalize_rho_advances(d)) {
    v.push_back({"finalize_rho", [d](cudaStream_t st) { return launch_finalize_rho_advance(d, st); }, 0, true});
  } else {
    v.push_back({"finalize_rho", [d](cudaStream_t st) { return launch_finalize_rho(d, 0, st); }, 0, true});
    v.push_back({"advance_iteration", [d](cudaStream_t st) { return launch_set_iteration(d, 0, 1, st); }});
  }
}

// after the polar of the M-step: P = M^T B (apply_m), rho_i^2 and the counter
// (finalize_rho).  With the cross term from the polar (polar_cross) rho_i^2 no
// longer waits for apply_m; on one rank the next E-step's tail_kk then runs on
// the side lane beside apply_m (early_kk).
void push_polar_tail(srm_plan* p, std::vector<Stage>& v) {
  const DevPlan& d = p->dp;
  if (!d.polar_cross) {
    v.push_back({"apply_m", [d](cudaStream_t st) { return launch_apply_m(d, 1, st); }});
    push_finalize_rho(d, v);
    return;
  }
  push_finalize_rho(d, v);
  if (p->early_kk) v.push_back({"tail_kk", [d](cudaStream_t st) { return launch_tail_kk(d, st); }, 1});
  v.push_back({"apply_m", [d](cudaStream_t st) { return launch_apply_m(d, 0, st); }});
}

// SRM_FLAG_EXACT_POLAR: M_i of local subjects [first, first + count) from A_i
// itself (TSQR levels, then the SVD of each R_i); RankError as kernels.py:202-206
cudaError_t launch_exact_polar(srm_plan* p, int first, int count, bool init, cudaStream_t st) {
  const QrJob* jobs = region<QrJob>(p, I_QRJOBS);
  cudaError_t e = cudaSuccess;
  for (size_t L = 0; L < p->qr.levels.size() && e == cudaSuccess; ++L) {
    int mx = 0;
    for (int i = first; i < first + count; ++i) mx = std::max(mx, p->qr.levels[L][i].nctas);
    e = launch_tsqr(jobs + (int64_t)L * p->n_local + first, count, mx, (int)p->K, st);
  }
  if (e == cudaSuccess)
    e = launch_svd_polar(region<SvdJob>(p, I_SVDJOBS) + first, count, (int)p->K, p->dp.status,
                         init ? nullptr : p->dp.iter, st);
  return e;
}

std::vector<Stage> m_stages(srm_plan* p) {
  const DevPlan& d = p->dp;
  std::vector<Stage> v;
  if (p->flags & SRM_FLAG_EXACT_POLAR) {
    v.push_back({"contract_a", [p, d](cudaStream_t st) {
                   return launch_contract_a((int)p->kp, p->dtype, d.xhat, p->ldx, d.S, p->ldx, p->ldx, d.amat, p->kp,
                                            0.5, region<ItemA>(p, I_ITEMS_A), (int)p->items_a.size(), st);
                 }});
    v.push_back({"contract_e_xhat", [p, d](cudaStream_t st) {
                   return launch_contract_e((int)p->kp, SRM_F64, p->dtype, d.amat, p->kp, d.xhat, p->ldx, d.part,
                                            p->ldo, 1.0, region<ItemE>(p, I_ITEMS_EX), (int)p->items_ex.size(), st);
                 }});
    v.push_back({"reduce_chunks", [d](cudaStream_t st) { return launch_reduce_chunks(d, st); }});
    v.push_back({"exact_polar", [p](cudaStream_t st) { return launch_exact_polar(p, 0, p->n_local, false, st); }});
    v.push_back({"apply_m", [d](cudaStream_t st) { return launch_apply_m(d, 1, st); }});
    push_finalize_rho(d, v);
    return v;
  }
  if (p->flags & SRM_FLAG_GRAM) {
    // B_i = S G_i / 2 straight into the reduced slot (G_i = X_i^T X_i, one-time)
    if (p->oz_sg) {
      // B_i = S G_i / 2 on the int8 tensor cores: slice S (rows), then one pass
      v.push_back({"oz_slice_s", [p, d](cudaStream_t st) {
                     return launch_oz_slice_rows(d.S, p->ldx, p->kp, p->ldx, region<int8_t>(p, I_OZS), p->oz_lqg,
                                                 region<int32_t>(p, I_OZSEXP), st);
                   }});
      // stream-K over all local subjects: every SM the same number of MMAs
      if (p->sk_off)
        v.push_back({"oz_sg", [p, d](cudaStream_t st) {
                       return launch_oz_sg(p->tm_g, p->tm_sq, region<int32_t>(p, I_OZGEXP),
                                           region<int32_t>(p, I_OZSEXP), d.bred, p->ldx, p->kp, p->ldo, 0, p->n_local,
                                           st);
                     }});
      else
      v.push_back({"oz_sg", [p, d](cudaStream_t st) {
                     return launch_oz_sg_sk(p->tm_g, p->tm_sq, region<int32_t>(p, I_OZGEXP),
                                            region<int32_t>(p, I_OZSEXP), d.bred, region<int32_t>(p, I_OZSKPART),
                                            region<int32_t>(p, I_OZSKFLAG), p->ldx, p->kp, p->ldo, 0, p->n_local,
                                            p->sk_ctas, st);
                   }});
    } else {
      v.push_back({"gram_b", [p, d](cudaStream_t st) {
                     return launch_contract_e((int)p->kp, SRM_F64, SRM_F64, d.st, p->kp, d.gram, p->ldx, d.bred,
                                              p->ldo, 0.5, region<ItemE>(p, I_ITEMS_BG), (int)p->items_bg.size(), st);
                   }});
    }
    v.push_back({"gram_from_b", [d](cudaStream_t st) { return launch_gram_from_b(d, st); }});
    v.push_back({"eig_polar", [d](cudaStream_t st) { return launch_eig_polar(d, 0, st); }});
    push_polar_tail(p, v);
    return v;
  }
  if (p->flags & SRM_FLAG_TC) {
    // fp32 X-hat on the tensor cores: A = X S^T / 2 and B = A^T X as 3xTF32
    v.push_back({"tc_apass", [p, d](cudaStream_t st) {
                   return launch_tc_apass(p->np, p->tm_x_a, p->tm_s, p->ldx, d.af, p->np, 0.5f,
                                          region<ItemA>(p, I_ITEMS_TA), (int)p->items_ta.size(), st);
                 }});
    v.push_back({"tc_bpass", [p, d](cudaStream_t st) {
                   return launch_tc_bpass(p->np, p->tm_a, p->tm_x_b, p->ldx, d.part, p->ldo, (int)p->kp,
                                          region<ItemE>(p, I_ITEMS_TB), (int)p->items_tb.size(), st);
                 }});
  } else {
  v.push_back({"contract_a", [p, d](cudaStream_t st) {
                 return launch_contract_a((int)p->kp, p->dtype, d.xhat, p->ldx, d.S, p->ldx, p->ldx, d.amat, p->kp,
                                          0.5, region<ItemA>(p, I_ITEMS_A), (int)p->items_a.size(), st);
               }});
  v.push_back({"contract_e_xhat", [p, d](cudaStream_t st) {
                 return launch_contract_e((int)p->kp, SRM_F64, p->dtype, d.amat, p->kp, d.xhat, p->ldx, d.part, p->ldo, 1.0,
                                          region<ItemE>(p, I_ITEMS_EX), (int)p->items_ex.size(), st);
               }});
  }
  v.push_back({"reduce_chunks", [d](cudaStream_t st) { return launch_reduce_chunks(d, st); }});
  v.push_back({"gram_from_b", [d](cudaStream_t st) { return launch_gram_from_b(d, st); }});
  v.push_back({"eig_polar", [d](cudaStream_t st) { return launch_eig_polar(d, 0, st); }});
  push_polar_tail(p, v);
  return v;
}

// Without `ln` every stage runs in order on `st`; with it, lane-1/2 stages run
// on the side streams (forked from `st` where they appear, unless fork is
// false: then they only follow their lane's earlier stages) and `st` waits
// for them at the next join stage and at the end of the list.  Graph capture
// turns the fork/join events into graph edges.
int run_stages(const std::vector<Stage>& stages, cudaStream_t st, const Lanes* ln = nullptr) {
  bool pending[3] = {false, false, false};
  for (const Stage& s : stages) {
    cudaStream_t target = st;
    cudaError_t e = cudaSuccess;
    if (ln && s.join)
      for (int l = 1; l <= 2 && e == cudaSuccess; ++l)
        if (pending[l]) {
          e = cudaStreamWaitEvent(st, ln->join[l], 0);
          pending[l] = false;
        }
    const int L = ln ? s.lane : 0;
    if (L > 0 && e == cudaSuccess) {
      if (s.fork) {
        e = cudaEventRecord(ln->fork[L], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ln->side[L], ln->fork[L], 0);
      }
      target = ln->side[L];
    }
    if (e == cudaSuccess) e = s.fn(target);
    if (L > 0 && e == cudaSuccess) {
      e = cudaEventRecord(ln->join[L], ln->side[L]);
      pending[L] = true;
    }
    if (e != cudaSuccess) return cuda_fail(e, s.name);
  }
  for (int l = 1; l <= 2; ++l)
    if (pending[l]) {
      cudaError_t e = cudaStreamWaitEvent(st, ln->join[l], 0);
      if (e != cudaSuccess) return cuda_fail(e, "join");
    }
  return SRM_OK;
}

int plan_lanes(srm_plan* p, const Lanes** out) {
  if (!p->lanes_ready) {
    for (int l = 1; l <= 2; ++l) {
      cudaError_t e = cudaStreamCreateWithFlags(&p->lanes.side[l], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->lanes.fork[l], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->lanes.join[l], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "side stream");
    }
    p->lanes_ready = true;
  }
  *out = &p->lanes;
  return SRM_OK;
}

int run_contractions(srm_plan* p, cudaStream_t st) {
  std::vector<Stage> v;
  contraction_stages(p, v);
  return run_stages(v, st);
}

std::vector<std::string> g_profile_names;

// one-time Gram X_i^T X_i of local subjects [first, first + count): int8
// slices on the tensor cores (SRM_FLAG_GRAM_I8) or fp64 DMMA tiles, then the
// lower triangle mirrored from the upper one
// model.W (srm.py:315-327): W_i = A_i M_i with M_i from the last M-step, for
// local subjects [first, first + count).  The shared prelude runs with the
// range that starts at subject 0; only the int8 W = Xhat R is split by
// subject (the other variants form every W_i in that first range).
// W = Xhat R over the final-W items [i0, i1): from the int8 records, or for fp32
// X-hat with the A operand sliced from X-hat in the kernel (ozw_x)
cudaError_t run_oz_w(srm_plan* p, const DevPlan& d, int i0, int i1, cudaStream_t st) {
  if (p->ozw_x)
    return launch_oz_wx(p->tm_xw, p->tm_r, region<int8_t>(p, I_OZR), region<int32_t>(p, I_OZEXP),
                        region<int32_t>(p, I_OZREXP), d.wout, region<OzItem>(p, I_ITEMS_OW) + i0, i1 - i0, p->ldx,
                        p->kp, p->K, st);
  return launch_oz_w(p->tm_q32, p->tm_r, region<int8_t>(p, I_OZR), region<int32_t>(p, I_OZREXP), d.wout,
                     region<OzItem>(p, I_ITEMS_OW) + i0, i1 - i0, p->ldx, p->kp, p->K, p->oz_nsl, st);
}

std::vector<Stage> finalize_stages(srm_plan* p, int first, int count) {
  const DevPlan& d = p->dp;
  std::vector<Stage> v;
  if (p->oz_w && first > 0) {
    const int i0 = p->ow_first[first], i1 = p->ow_first[first + count];
    v.push_back({"oz_w", [p, d, i0, i1](cudaStream_t st) { return run_oz_w(p, d, i0, i1, st); }});
    return v;
  }
  if (first > 0) return v;
  if (p->oz_w) {
    // W_i = Xhat_i R_i, R_i = S^T M_i / 2, from the int8 slices of Xhat on the
    // tensor cores (no A pass, no W = A M pass)
    v.push_back({"oz_rt", [p, d](cudaStream_t st) {
                   return launch_oz_rt(d.mmat, d.S, region<int32_t>(p, I_OZEXP), d.part, p->ldx, p->kp, p->K,
                                       p->n_local, st);
                 }});
    v.push_back({"oz_slice_r", [p, d](cudaStream_t st) {
                   return launch_oz_slice_rows(d.part, p->ldx, (int64_t)p->n_local * p->kp, p->ldx,
                                               region<int8_t>(p, I_OZR), p->oz_lqg, region<int32_t>(p, I_OZREXP), st,
                                               -p->kp);
                 }});
    const int i1 = p->ow_first[count];
    v.push_back({"oz_w", [p, d, i1](cudaStream_t st) { return run_oz_w(p, d, 0, i1, st); }});
    return v;
  }
  if (p->flags & SRM_FLAG_GRAM) {  // A_i = Xhat_i S^T / 2 is not kept per iteration on the Gram path
    v.push_back({"final_a", [p, d](cudaStream_t st) {
                   return launch_contract_a((int)p->kp, p->dtype, d.xhat, p->ldx, d.S, p->ldx, p->ldx, d.amat, p->kp,
                                            0.5, region<ItemA>(p, I_ITEMS_A), (int)p->items_a.size(), st);
                 }});
  }
  if (p->flags & SRM_FLAG_TC) {
    // W = A M with M from the exact fp64 Gram of the stored fp32 A, so the
    // returned W is orthonormal to fp64 precision (acceptance criterion 4)
    // even though the per-iteration passes run in 3xTF32
    v.push_back({"final_gram", [p, d](cudaStream_t st) {
                   return launch_contract_e((int)p->kp, SRM_F32, SRM_F32, d.af, p->np, d.af, p->np, d.part, p->ldo,
                                            1.0, region<ItemE>(p, I_ITEMS_TG), (int)p->items_tg.size(), st);
                 }});
    v.push_back({"final_reduce", [d](cudaStream_t st) { return launch_reduce_chunks(d, st); }});
    // the final transform goes to its own buffer (QSCR): MMAT still holds the
    // iteration's M, which the next iteration's apply_m reads when a caller
    // forms W mid-fit (on_iteration snapshots, rotated iteration graph)
    DevPlan fd = d;
    fd.mmat = region<double>(p, I_QSCR);
    v.push_back({"final_polar", [fd](cudaStream_t st) { return launch_final_polar(fd, st); }});
    v.push_back({"apply_w", [p, fd](cudaStream_t st) {
                   return launch_apply_rows((int)p->kp, SRM_F32, fd.af, p->np, fd.mmat, p->kp * p->kp, fd.wout,
                                            (int)p->K, region<ItemA>(p, I_ITEMS_TA), (int)p->items_ta.size(), st);
                 }});
    return v;
  }
  v.push_back({"apply_w", [p, d](cudaStream_t st) {
                 return launch_apply_rows((int)p->kp, SRM_F64, d.amat, p->kp, d.mmat, p->kp * p->kp, d.wout,
                                          (int)p->K, region<ItemA>(p, I_ITEMS_A), (int)p->items_a.size(), st);
               }});
  return v;
}

std::vector<Stage> gram_stages(srm_plan* p, int first, int count) {
  const DevPlan& d = p->dp;
  std::vector<Stage> v;
  if (p->flags & SRM_FLAG_GRAM_I8) {
    const int per = (int)(p->items_oz.size() / p->n_local);  // upper tiles per subject (subject-major)
    v.push_back({"oz_split", [p, d, first, count](cudaStream_t st) {
                   return launch_oz_prepare(d, p->dtype, p->oz_nsl, first, count,
                                            region<unsigned long long>(p, I_OZCMAX), region<int8_t>(p, I_OZQ),
                                            p->oz_lq, region<int32_t>(p, I_OZEXP), p->max_v, st);
                 }});
    const OzGramOut o{d.gram, p->ldx, p->ldx * p->ldx, p->ldx, region<int32_t>(p, I_OZEXP), p->ldx, p->ldx, p->T};
    if (!p->items_oz2.empty()) {
      // the CTA-pair tiles (the batched prepare runs them beside the single tiles)
      const int per2 = (int)(p->items_oz2.size() / p->n_local);
      v.push_back({"oz_gram_pairs", [p, o, first, count, per2](cudaStream_t st) {
                     return launch_oz_gram2(p->tm_q, p->tm_qb, o, region<OzItem>(p, I_ITEMS_OZ2) + (int64_t)first * per2,
                                            count * per2, p->oz_nsl, st);
                   }});
    }
    v.push_back({"oz_gram", [p, o, first, count, per](cudaStream_t st) {
                   return launch_oz_gram(p->tm_q, o, region<OzItem>(p, I_ITEMS_OZ) + (int64_t)first * per,
                                         count * per, p->oz_nsl, st);
                 }});
  } else {
    const int per = (int)(p->items_gram.size() / p->n_local);
    v.push_back({"gram_tiles", [p, d, first, count, per](cudaStream_t st) {
                   return launch_gram_tiles(p->dtype, d.xhat, p->ldx, d.gram, p->ldx,
                                            region<ItemE>(p, I_ITEMS_GRAM) + (int64_t)first * per, count * per, st);
                 }});
  }
  v.push_back({"mirror_gram", [d, first, count](cudaStream_t st) { return launch_mirror_gram(d, first, count, st); }});
  if (p->oz_sg) {
    // row slices of G_i for the per-iteration int8 B = S G / 2
    v.push_back({"oz_slice_g", [p, d, first, count](cudaStream_t st) {
                   return launch_oz_slice_rows(d.gram + (int64_t)first * p->ldx * p->ldx, p->ldx,
                                               (int64_t)count * p->ldx, p->ldx,
                                               region<int8_t>(p, I_OZG) + (int64_t)first * (int64_t)oz_tiled_bytes(p->ldx, p->ldx),
                                               p->oz_lqg, region<int32_t>(p, I_OZGEXP) + (int64_t)first * p->ldx, st,
                                               p->ldx);
                 }});
  }
  return v;
}

// run stages eagerly with an event between kernels; names -> srm_profile_name
int profile_stages(const std::vector<Stage>& stages, float* ms_out, int capacity, int* n_out, cudaStream_t st) {
  const int n = (int)stages.size();
  std::vector<cudaEvent_t> ev(n + 1);
  for (auto& e : ev) cudaEventCreate(&e);
  cudaEventRecord(ev[0], st);
  int rc = SRM_OK;
  for (int i = 0; i < n && rc == SRM_OK; ++i) {
    cudaError_t e = stages[i].fn(st);
    if (e != cudaSuccess) rc = cuda_fail(e, stages[i].name);
    cudaEventRecord(ev[i + 1], st);
  }
  cudaError_t e = cudaEventSynchronize(ev[n]);
  if (rc == SRM_OK && e != cudaSuccess) rc = cuda_fail(e, "profile sync");
  g_profile_names.clear();
  for (int i = 0; i < n; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
    if (i < capacity) ms_out[i] = ms;
    g_profile_names.push_back(stages[i].name);
  }
  for (auto& x : ev) cudaEventDestroy(x);
  *n_out = n;
  return rc;
}


}  // namespace

extern "C" {

int srm_abi_version(void) { return SRM_B200_ABI_VERSION; }

const char* srm_last_error(void) { return g_last_error.c_str(); }

int srm_plan_create(srm_plan** out, int dtype, int n_local, const int64_t* n_voxels, int64_t n_trs,
                    int64_t k, int iterations, int world_size, int rank,
                    const int32_t* counts_per_rank, int flags) {
  if (!out) return fail(SRM_ERR_CONFIG, "null plan pointer");
  *out = nullptr;
  if (dtype != SRM_F64 && dtype != SRM_F32) return fail(SRM_ERR_CONFIG, "dtype must be SRM_F64 or SRM_F32");
  if (k < 1) return fail(SRM_ERR_CONFIG, "k must be at least 1");
  if (iterations < 1) return fail(SRM_ERR_CONFIG, "iterations must be at least 1");
  if (n_local < 1) return fail(SRM_ERR_CONFIG, "each worker needs at least one subject");
  if (n_trs < 1) return fail(SRM_ERR_SHAPE, "need at least 1 TR");
  if (k > max_supported_k())
    return fail(SRM_ERR_UNSUPPORTED, "k > " + std::to_string(max_supported_k()) + " is not supported by this build");
  if (world_size < 1 || rank < 0 || rank >= world_size) return fail(SRM_ERR_CONFIG, "invalid rank/size");
  if (!counts_per_rank) return fail(SRM_ERR_CONFIG, "counts_per_rank is required");
  if (counts_per_rank[rank] != n_local) return fail(SRM_ERR_CONFIG, "counts_per_rank[rank] != n_local");
  srm_plan* p = new srm_plan();
  p->dtype = dtype;
  p->n_local = n_local;
  p->V.assign(n_voxels, n_voxels + n_local);
  for (int i = 0; i < n_local; ++i) {
    if (p->V[i] < k) {
      delete p;
      return fail(SRM_ERR_SHAPE, "subject has " + std::to_string(n_voxels[i]) + " voxels, fewer than k=" +
                                     std::to_string(k) + " factors");
    }
  }
  p->T = n_trs;
  p->K = k;
  p->kp = round_up(k, 8);
  p->ldx = round_up(n_trs, 32);
  p->ldo = p->ldx + p->kp;
  p->iterations = iterations;
  p->world = world_size;
  p->rank = rank;
  p->counts.assign(counts_per_rank, counts_per_rank + world_size);
  p->flags = flags;
  if (world_size == 1) p->flags |= SRM_FLAG_ORDERED;
  // column-block exchange: multi-rank only; it replaces the gathered table
  if (p->flags & SRM_FLAG_COLBLOCK) p->flags &= world_size > 1 ? ~SRM_FLAG_ORDERED : ~SRM_FLAG_COLBLOCK;
  if ((p->flags & SRM_FLAG_TC) && (dtype != SRM_F32 || !tc_supported((int)k))) p->flags &= ~SRM_FLAG_TC;
  if ((p->flags & SRM_FLAG_TC) && (p->flags & SRM_FLAG_GRAM)) p->flags &= ~SRM_FLAG_TC;
  if ((p->flags & SRM_FLAG_GRAM_I8) && !(p->flags & SRM_FLAG_GRAM)) p->flags &= ~SRM_FLAG_GRAM_I8;
  if (p->flags & SRM_FLAG_EXACT_POLAR) {
    // A_i is formed every iteration (fp64 streaming path) so its own QR/SVD gives M_i
    p->flags &= ~(SRM_FLAG_GRAM | SRM_FLAG_GRAM_I8 | SRM_FLAG_TC);
    if (!qr_polar_supported((int)k)) {
      delete p;
      return fail(SRM_ERR_UNSUPPORTED, "k = " + std::to_string(k) + " exceeds the exact polar route's shared memory");
    }
  }
  p->np = tc_np((int)k);
  p->n_total = 0;
  p->max_local = 0;
  p->global0 = 0;
  for (int r = 0; r < world_size; ++r) {
    if (r < rank) p->global0 += p->counts[r];
    p->n_total += p->counts[r];
    p->max_local = std::max(p->max_local, p->counts[r]);
  }
  if (p->flags & SRM_FLAG_ORDERED) {
    p->n_slots = world_size * p->max_local;
    p->slot0 = rank * p->max_local;
  } else {
    p->n_slots = n_local;
    p->slot0 = 0;
  }
  p->row_off.assign(n_local, 0);
  int64_t r = 0;
  for (int i = 0; i < n_local; ++i) {
    p->row_off[i] = r;
    r += p->V[i];
  }
  p->rows_total = r;
  build_work(p);
  layout(p);
  p->sliced.assign(n_local, 0);
  *out = p;
  return SRM_OK;
}

int srm_plan_destroy(srm_plan* plan) {
  if (plan) {
    if (plan->graph_exec) cudaGraphExecDestroy(plan->graph_exec);
    if (plan->graph) cudaGraphDestroy(plan->graph);
    if (plan->cap_stream) cudaStreamDestroy(plan->cap_stream);
    if (plan->lanes_ready)
      for (int l = 1; l <= 2; ++l) {
        cudaStreamDestroy(plan->lanes.side[l]);
        cudaEventDestroy(plan->lanes.fork[l]);
        cudaEventDestroy(plan->lanes.join[l]);
      }
    for (cudaEvent_t ev : plan->gram_events) cudaEventDestroy(ev);
    for (cudaEvent_t ev : plan->post_events) cudaEventDestroy(ev);
    if (plan->hi_stream) cudaStreamDestroy(plan->hi_stream);
    if (plan->hi_stream2) cudaStreamDestroy(plan->hi_stream2);
    for (cudaEvent_t ev : plan->pair_events) cudaEventDestroy(ev);
  }
  delete plan;
  return SRM_OK;
}

int64_t srm_plan_workspace_bytes(const srm_plan* plan) { return plan ? plan->total_bytes : -1; }

int64_t srm_plan_dim(const srm_plan* p, int which) {
  if (!p) return -1;
  switch (which) {
    case SRM_D_LDX: return p->ldx;
    case SRM_D_KP: return p->kp;
    case SRM_D_ROWS: return p->rows_total;
    case SRM_D_TERM_STRIDE: return p->dp.term_stride;
    case SRM_D_RED_STRIDE: return p->dp.red_stride;
    case SRM_D_HIST_STRIDE: return p->dp.hist_stride;
    case SRM_D_N_SLOTS: return p->n_slots;
    case SRM_D_SLOT_OFFSET: return p->slot0;
    case SRM_D_ITEMS_E: return (int64_t)(p->items_ex.size() + p->items_ea.size());
    case SRM_D_ITEMS_A: return (int64_t)p->items_a.size();
    case SRM_D_CHUNK_ROWS: return p->chunk_rows;
    case SRM_D_FLAGS: return p->flags;
    case SRM_D_XREC: return p->kp * ((p->ldx + p->world - 1) / p->world) + kRecScalars;
    case SRM_D_XRED: return p->kp * ((p->ldx + p->world - 1) / p->world) + kRedScalars;
    case SRM_D_LAUNCHES: return (int64_t)(e_stages(const_cast<srm_plan*>(p)).size() + m_stages(const_cast<srm_plan*>(p)).size());
    default: return -1;
  }
}

int srm_plan_region(const srm_plan* p, int region_id, int64_t* offset, int64_t* bytes) {
  if (!p || region_id < 0 || region_id >= SRM_R_COUNT) return fail(SRM_ERR_CONFIG, "bad region");
  if (offset) *offset = p->off[region_id];
  if (bytes) *bytes = p->size[region_id];
  return SRM_OK;
}

int srm_plan_bind(srm_plan* p, void* workspace, int64_t bytes) {
  if (!p || !workspace) return fail(SRM_ERR_CONFIG, "null plan/workspace");
  if (bytes < p->total_bytes) return fail(SRM_ERR_CONFIG, "workspace too small");
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0) return fail(SRM_ERR_CONFIG, "workspace must be 256-byte aligned");
  p->ws = static_cast<char*>(workspace);
  set_pointers(p);
  // zero everything except the bulk regions every fit writes in full before
  // reading them (X-hat by srm_load_subject, G and the int8 slices by
  // srm_prepare_gram): tens of GB that need no clearing
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < I_COUNT && e == cudaSuccess; ++r) {
    if (r == SRM_R_XHAT || r == SRM_R_GRAM || r == I_OZQ || p->size[r] == 0) continue;
    e = cudaMemsetAsync(p->ws + p->off[r], 0, round_up(p->size[r], 256), 0);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  if (e != cudaSuccess) return cuda_fail(e, "bind memset");
  struct Up {
    int r;
    const void* src;
  } ups[] = {{I_SUBJ, p->subj.data()},         {I_ORDER, p->order.data()},
             {I_ORDER_LOCAL, p->order_local.data()}, {I_ITEMS_EX, p->items_ex.data()},
             {I_ITEMS_EA, p->items_ea.data()},  {I_ITEMS_A, p->items_a.data()},
             {I_ITEMS_GRAM, p->items_gram.data()},
             {I_ITEMS_BG, p->items_bg.data()},   {I_ITEMS_TB, p->items_tb.data()},
             {I_ITEMS_TA, p->items_ta.data()},   {I_ITEMS_TG, p->items_tg.data()},
             {I_ITEMS_OZ, p->items_oz.data()},   {I_ITEMS_OW, p->items_ow.data()},
             {I_ITEMS_TN, p->items_tn.data()},   {I_ITEMS_GG, p->items_gg.data()},
             {I_ITEMS_OZ2, p->items_oz2.data()},  {I_XCOUNTS, p->counts.data()}};
  for (const Up& u : ups) {
    if (p->size[u.r] == 0) continue;
    e = cudaMemcpy(p->ws + p->off[u.r], u.src, p->size[u.r], cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "bind upload");
  }
  if (p->flags & SRM_FLAG_EXACT_POLAR) {
    std::vector<const double*> a;
    std::vector<int64_t> lda;
    for (int i = 0; i < p->n_local; ++i) {
      a.push_back(region<double>(p, SRM_R_AMAT) + p->row_off[i] * p->kp);
      lda.push_back(p->kp);
    }
    std::vector<const double*> rfin;
    const auto lv = tsqr_jobs(p->qr, a, lda, (int)p->K, region<double>(p, I_QRBUF0), region<double>(p, I_QRBUF1), &rfin);
    std::vector<QrJob> flat;
    for (const auto& l : lv) flat.insert(flat.end(), l.begin(), l.end());
    std::vector<SvdJob> sv;
    for (int i = 0; i < p->n_local; ++i)
      sv.push_back({rfin[i], region<double>(p, SRM_R_MMAT) + (int64_t)i * p->kp * p->kp, p->kp, (int32_t)p->kp,
                    (int32_t)(p->global0 + i),
                    svd_needs_global_v((int)p->K) ? region<double>(p, I_QSCR) + (int64_t)i * p->kp * p->kp : nullptr});
    e = cudaMemcpy(region<QrJob>(p, I_QRJOBS), flat.data(), flat.size() * sizeof(QrJob), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(region<SvdJob>(p, I_SVDJOBS), sv.data(), sv.size() * sizeof(SvdJob), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "bind qr jobs");
  }
  // Sigma_s = I (srm.py:248); S starts at zero
  std::vector<double> eye((size_t)p->kp * p->kp, 0.0);
  for (int64_t j = 0; j < p->K; ++j) eye[(size_t)j * p->kp + j] = 1.0;
  e = cudaMemcpy(region<double>(p, SRM_R_SIGMA), eye.data(), eye.size() * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "bind sigma");
  // its inverse as k_tail_inv leaves it (-I; log det 0 from the memset)
  for (double& x : eye) x = -x;
  e = cudaMemcpy(region<double>(p, I_SINV), eye.data(), eye.size() * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "bind sigma inverse");
  // warm up kernel attributes outside any graph capture
  const DevPlan& d = p->dp;
  e = launch_contract_e((int)p->kp, SRM_F64, p->dtype, d.amat, p->kp, d.xhat, p->ldx, d.part, p->ldo, 1.0, nullptr, 0, 0);
  if (e == cudaSuccess)
    e = launch_contract_e((int)p->kp, SRM_F64, SRM_F64, d.amat, p->kp, d.amat, p->kp, d.part, p->ldo, 1.0, nullptr, 0, 0);
  if (e == cudaSuccess)
    e = launch_contract_a((int)p->kp, p->dtype, d.xhat, p->ldx, d.S, p->ldx, p->ldx, d.amat, p->kp, 0.5, nullptr, 0, 0);
  if (e == cudaSuccess)
    e = launch_contract_a((int)p->kp, SRM_F64, d.bred, p->ldo, d.S, p->ldx, p->ldx, d.bred, p->ldo, 0.5, nullptr, 0, 0);
  if (e == cudaSuccess && (p->flags & SRM_FLAG_TC))
    e = launch_contract_e((int)p->kp, SRM_F32, SRM_F32, d.af, p->np, d.af, p->np, d.part, p->ldo, 1.0, nullptr, 0, 0);
  if (e == cudaSuccess && (p->flags & SRM_FLAG_TC)) {
    const float* xf = static_cast<const float*>(d.xhat);
    e = make_map_f32(&p->tm_x_a, xf, p->ldx, p->rows_total, p->ldx, 32, 256, true);
    if (e == cudaSuccess) e = make_map_f32(&p->tm_s, d.sf, p->ldx, 2 * p->np, p->ldx, 32, p->np, true);
    if (e == cudaSuccess) e = make_map_f32(&p->tm_a, d.af, p->np, p->rows_total, p->np, p->np, 32, false);
    if (e == cudaSuccess) e = make_map_f32(&p->tm_x_b, xf, p->ldx, p->rows_total, p->ldx, 256, 32, false);
    if (e != cudaSuccess) return cuda_fail(e, "tensor maps");
    e = launch_tc_apass(p->np, p->tm_x_a, p->tm_s, p->ldx, d.af, p->np, 0.5f, nullptr, 0, 0);
    if (e == cudaSuccess) e = launch_tc_bpass(p->np, p->tm_a, p->tm_x_b, p->ldx, d.part, p->ldo, (int)p->kp, nullptr, 0, 0);
  }
  if (e == cudaSuccess && (p->flags & SRM_FLAG_GRAM))
    e = launch_gram_tiles(p->dtype, d.xhat, p->ldx, d.gram, p->ldx, nullptr, 0, 0);
  if (e == cudaSuccess && (p->flags & SRM_FLAG_GRAM_I8)) {
    e = make_map_q(&p->tm_q, region<int8_t>(p, I_OZQ), p->oz_lq, p->ldx, p->n_local, 128);
    if (e == cudaSuccess) e = make_map_q(&p->tm_qb, region<int8_t>(p, I_OZQ), p->oz_lq, p->ldx, p->n_local, 64);
    const OzGramOut none{};
    if (e == cudaSuccess) e = launch_oz_gram(p->tm_q, none, nullptr, 0, p->oz_nsl, 0);
    if (e == cudaSuccess) e = launch_oz_gram(p->tm_q, none, nullptr, 0, 7, 0);
    if (e == cudaSuccess) e = launch_oz_gram2(p->tm_q, p->tm_qb, none, nullptr, 0, p->oz_nsl, 0);
    if (e == cudaSuccess && p->oz_sg) {
      // tiled G slices: rows of 128 B, oz_tiled_bytes / 128 rows per subject
      e = make_map_q(&p->tm_g, region<int8_t>(p, I_OZG), 128, (int64_t)oz_tiled_bytes(p->ldx, p->ldx) / 128,
                     p->n_local, 128);
      if (e == cudaSuccess) e = make_map_q8(&p->tm_sq, region<int8_t>(p, I_OZS), p->oz_lqg, p->kp, 1);
      if (e == cudaSuccess)
        e = launch_oz_sg(p->tm_g, p->tm_sq, nullptr, nullptr, nullptr, p->ldx, p->kp, p->ldo, 0, 0, 0);
      if (e == cudaSuccess)
        e = launch_oz_sg_sk(p->tm_g, p->tm_sq, nullptr, nullptr, nullptr, nullptr, nullptr, p->ldx, p->kp, p->ldo, 0, 0,
                            p->sk_ctas, 0);
    }
    if (e == cudaSuccess && p->oz_lqg_init) {
      e = make_map_q(&p->tm_gi, region<int8_t>(p, SRM_R_WOUT), p->oz_lqg_init, p->K, p->n_local, 128);
      if (e == cudaSuccess)
        // (k_oz_nt: the draw's slots of a voxel block slot-major, eight or -- four-slice X-hat,
        // d-groups 0-3 -- the four it reads)
        e = make_map_q8(&p->tm_gi64, region<int8_t>(p, SRM_R_WOUT), p->oz_lqg_init, p->K, p->n_local,
                        p->oz_nsl == 4 ? 4 : 8);
      if (e == cudaSuccess)
        e = launch_oz_tn(p->tm_gi, p->tm_q, nullptr, nullptr, nullptr, p->ldx, p->kp, p->ldo, p->K, nullptr, 0,
                         p->oz_nsl, 0);
      if (e == cudaSuccess)
        e = launch_oz_nt(p->tm_q, p->tm_gi64, nullptr, nullptr, nullptr, p->ldx, p->kp, p->ldo, p->K, nullptr, 0,
                         p->oz_nsl, 0);
    }
    if (e == cudaSuccess && p->oz_w) {
      e = make_map_q5(&p->tm_q32, region<int8_t>(p, I_OZQ), p->oz_lq, p->ldx, p->n_local, p->oz_nsl);
      // four-slice X-hat: the final W keeps d-groups 0-4, which read R's slots 0-5 only
      if (e == cudaSuccess)
        e = make_map_q8(&p->tm_r, region<int8_t>(p, I_OZR), p->oz_lqg, p->kp, p->n_local, p->oz_nsl == 4 ? 6 : 8);
      if (e == cudaSuccess)
        e = launch_oz_w(p->tm_q32, p->tm_r, nullptr, nullptr, nullptr, nullptr, 0, p->ldx, p->kp, p->K, p->oz_nsl, 0);
      if (e == cudaSuccess && p->ozw_x) {
        e = make_map_f32(&p->tm_xw, static_cast<const float*>(d.xhat), p->ldx, p->rows_total, p->ldx, 32, 128, true);
        if (e == cudaSuccess)
          e = launch_oz_wx(p->tm_xw, p->tm_r, nullptr, nullptr, nullptr, nullptr, nullptr, 0, p->ldx, p->kp, p->K, 0);
      }
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "kernel attributes");
  return SRM_OK;
}

int srm_load_subject(srm_plan* p, int local, const void* x, int x_dtype, int64_t ld, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  if (local < 0 || local >= p->n_local) return fail(SRM_ERR_CONFIG, "subject index out of range");
  if (x_dtype != SRM_F64 && x_dtype != SRM_F32) return fail(SRM_ERR_CONFIG, "x dtype must be f64 or f32");
  if (ld < p->T) return fail(SRM_ERR_SHAPE, "leading dimension smaller than T");
  return check(launch_prep(p->dp, local, p->V[local], x, x_dtype, ld, p->dtype, as_stream(stream)), "prep");
}

int srm_finish_load(srm_plan* p, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  return check(launch_subject_sqnorm(p->dp, as_stream(stream)), "sqnorm");
}

int srm_init_mapping_range(srm_plan* p, int first, int count, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  if (first < 0 || count < 0 || first + count > p->n_local) return fail(SRM_ERR_CONFIG, "subject range out of bounds");
  if (count == 0) return SRM_OK;
  cudaStream_t st = as_stream(stream);
  DevPlan d = p->dp;
  d.sub0 = first;
  d.nsub = count;
  // the split-V items are subject-major: nchunk[i] x (ldx / 128) tiles (ex) and nchunk[i] (ea) per subject
  const int64_t ntiles = (p->ldx + 127) / 128;
  int64_t ex0 = 0, exn = 0, ean = 0;
  for (int i = 0; i < first; ++i) ex0 += p->nchunk[i] * ntiles;
  for (int i = first; i < first + count; ++i) {
    exn += p->nchunk[i] * ntiles;
    ean += p->nchunk[i];
  }
  const bool exact = (p->flags & SRM_FLAG_EXACT_POLAR) != 0;
  // B_0 = G^T Xhat: on int8 Gram plans from the slices of G and of Xhat (the
  // caller has run srm_prepare_gram_range over these subjects), after the
  // chunk reduction of G^T G; otherwise one more split-V DMMA contraction
  const bool i8 = p->oz_lqg_init != 0;
  // kp > 64: the draw's A^T A from its slices as well (k_oz_gram on one
  // diagonal tile per V chunk), after launch_oz_init_slices below
  const bool gg_i8 = i8 && !exact && !p->items_gg.empty();
  cudaError_t e = cudaSuccess;
  if (!i8)
    e = launch_contract_e((int)p->kp, SRM_F64, p->dtype, d.amat, p->kp, d.xhat, p->ldx, d.part, p->ldo, 1.0,
                          region<ItemE>(p, I_ITEMS_EX) + ex0, (int)exn, st);
  if (e == cudaSuccess && !exact && !gg_i8)  // the Gram route's A^T A of the draw
    e = launch_contract_e((int)p->kp, SRM_F64, SRM_F64, d.amat, p->kp, d.amat, p->kp, d.part, p->ldo, 1.0,
                          region<ItemE>(p, I_ITEMS_EA) + p->chunk0[first], (int)ean, st);
  if (e == cudaSuccess && !gg_i8) e = launch_reduce_chunks(d, st);
  if (e == cudaSuccess && i8) {
    // Xhat's slices must exist: prepare subjects no srm_prepare_gram_range call
    // has covered yet (stream order; the loader already does it on this stream)
    for (int i = first; i < first + count; ++i)
      if (!p->sliced[i]) {
        const int rc = srm_prepare_gram_range(p, i, 1, stream);
        if (rc) return rc;
      }
    int64_t maxv = 0;
    for (int i = first; i < first + count; ++i) maxv = std::max(maxv, p->V[i]);
    e = launch_oz_init_slices(d, first, count, region<int8_t>(p, SRM_R_WOUT), p->oz_lqg_init,
                              region<int32_t>(p, I_OZGIEXP), region<unsigned long long>(p, I_OZGICMAX), maxv, st);
    if (e == cudaSuccess && gg_i8) {
      // partial A^T A of chunk c at part[c][0..kp)[ldx..ldx + kp), as the DMMA items write it
      const OzGramOut o{d.part + p->ldx, p->ldo, p->kp * p->ldo, p->kp, region<int32_t>(p, I_OZGIEXP), p->K, p->K,
                        p->K};
      e = launch_oz_gram(p->tm_gi, o, region<OzItem>(p, I_ITEMS_GG) + p->chunk0[first], (int)ean, 7, st);
      if (e == cudaSuccess) e = launch_reduce_chunks(d, st);
    }
    const int per = (int)((p->ldx + 127) / 128);
    // kp <= 64: the transposed one-pass kernel (N = 64 features); else M = 128 features
    static const bool nt_off = [] {
      const char* v = getenv("SRM_B200_INIT_NT");
      return v && v[0] == '0';
    }();
    if (e == cudaSuccess && p->kp <= 64 && !nt_off)
      e = launch_oz_nt(p->tm_q, p->tm_gi64, region<int32_t>(p, I_OZGIEXP), region<int32_t>(p, I_OZEXP), d.bred,
                       p->ldx, p->kp, p->ldo, p->K, region<OzItem>(p, I_ITEMS_TN) + (int64_t)first * per, count * per,
                       p->oz_nsl, st);
    else if (e == cudaSuccess)
      e = launch_oz_tn(p->tm_gi, p->tm_q, region<int32_t>(p, I_OZGIEXP), region<int32_t>(p, I_OZEXP), d.bred, p->ldx,
                       p->kp, p->ldo, p->K, region<OzItem>(p, I_ITEMS_TN) + (int64_t)first * per, count * per,
                       p->oz_nsl, st);
  }
  if (e == cudaSuccess) e = exact ? launch_exact_polar(p, first, count, true, st) : launch_eig_polar(d, 1, st);
  if (e == cudaSuccess) e = launch_apply_m(d, 0, st);
  if (e == cudaSuccess) e = launch_finalize_rho(d, 1, st);
  // early_kk: the first E-step's K x K tail once every rho_i^2 = 1 is in place
  if (e == cudaSuccess && p->early_kk && first + count == p->n_local) e = launch_tail_kk(p->dp, st);
  return check(e, "init_mapping");
}

int srm_init_mapping(srm_plan* p, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  const int rc = srm_init_mapping_range(p, 0, p->n_local, stream);
  if (rc) return rc;
  return check(launch_set_iteration(p->dp, 0, 0, as_stream(stream)), "init_mapping");
}

int srm_xchg_pack(srm_plan* p, void* stream) {
  if (!p || !p->ws || !(p->flags & SRM_FLAG_COLBLOCK)) return fail(SRM_ERR_CONFIG, "not a column-block plan");
  return check(launch_xchg_pack(p->dp, as_stream(stream)), "xchg_pack");
}

int srm_xchg_reduce(srm_plan* p, void* stream) {
  if (!p || !p->ws || !(p->flags & SRM_FLAG_COLBLOCK)) return fail(SRM_ERR_CONFIG, "not a column-block plan");
  return check(launch_xchg_reduce(p->dp, as_stream(stream)), "xchg_reduce");
}

int srm_xchg_unpack(srm_plan* p, void* stream) {
  if (!p || !p->ws || !(p->flags & SRM_FLAG_COLBLOCK)) return fail(SRM_ERR_CONFIG, "not a column-block plan");
  return check(launch_xchg_unpack(p->dp, as_stream(stream)), "xchg_unpack");
}

int srm_reduce_local(srm_plan* p, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  return check(launch_reduce_terms(p->dp, p->dp.redlocal, region<int32_t>(p, I_ORDER_LOCAL), p->n_local,
                                   as_stream(stream)),
               "reduce_local");
}

int srm_set_iteration(srm_plan* p, int iteration, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  if (iteration < 0) return fail(SRM_ERR_CONFIG, "iteration must be >= 0");
  return check(launch_set_iteration(p->dp, iteration, 0, as_stream(stream)), "set_iteration");
}

int srm_e_step(srm_plan* p, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  const Lanes* ln = nullptr;
  const int rc = plan_lanes(p, &ln);
  if (rc) return rc;
  return run_stages(e_stages(p), as_stream(stream), ln);
}

int srm_m_step(srm_plan* p, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  return run_stages(m_stages(p), as_stream(stream));
}

// The stages of one captured EM iteration.  With early_kk the M-step ends
// with {tail_kk (side lane) || apply_m} after finalize_rho, and a graph replay
// joins every lane at its end -- so the captured iteration is rotated to
// [tail_kk || apply_m] [E-step] [M-step up to finalize_rho]: the next E-step's
// reduce_terms then follows apply_m inside the same graph while tail_kk runs,
// and the lanes meet at finalize_rho (which waits for tail_sigma anyway).
// Replays compose to the eager order E M E M ...; the first replay repeats the
// init's own apply_m and tail_kk (the same inputs, so the same values).
std::vector<Stage> iteration_stages(srm_plan* p) {
  std::vector<Stage> e = e_stages(p), m = m_stages(p);
  size_t cut = m.size();
  if (p->early_kk)
    for (size_t k = 0; k < m.size(); ++k)
      if (!strcmp(m[k].name, "finalize_rho") || !strcmp(m[k].name, "advance_iteration")) cut = k + 1;
  std::vector<Stage> v(m.begin() + cut, m.end());
  v.insert(v.end(), e.begin(), e.end());
  v.insert(v.end(), m.begin(), m.begin() + cut);
  return v;
}

int srm_graph_capture(srm_plan* p) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  if (p->graph_exec) return SRM_OK;
  cudaError_t e = cudaSuccess;
  if (!p->cap_stream) e = cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e, "capture stream");
  e = cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_fail(e, "begin capture");
  // one list: the side-stream stages of the E-step overlap the M-step
  std::vector<Stage> stages = iteration_stages(p);
  const Lanes* ln = nullptr;
  int rc = plan_lanes(p, &ln);
  if (rc == SRM_OK) rc = run_stages(stages, p->cap_stream, ln);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(p->cap_stream, &g);
  if (rc != SRM_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return cuda_fail(e, "end capture");
  e = cudaGraphInstantiate(&p->graph_exec, g, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    return cuda_fail(e, "instantiate");
  }
  p->graph = g;
  return SRM_OK;
}

int srm_graph_launch(srm_plan* p, void* stream) {
  if (!p || !p->graph_exec) return fail(SRM_ERR_CONFIG, "no captured graph");
  return check(cudaGraphLaunch(p->graph_exec, as_stream(stream)), "graph launch");
}

int srm_profile_iteration(srm_plan* p, float* ms_out, int capacity, int* n_out, void* stream) {
  if (!p || !p->ws || !ms_out || !n_out) return fail(SRM_ERR_CONFIG, "plan not bound");
  std::vector<Stage> stages = e_stages(p);
  std::vector<Stage> m = m_stages(p);
  stages.insert(stages.end(), m.begin(), m.end());
  return profile_stages(stages, ms_out, capacity, n_out, as_stream(stream));
}

const char* srm_profile_name(int index) {
  if (index < 0 || index >= (int)g_profile_names.size()) return "";
  return g_profile_names[index].c_str();
}

int srm_finalize(srm_plan* p, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  return run_stages(finalize_stages(p, 0, p->n_local), as_stream(stream));
}

int srm_finalize_range(srm_plan* p, int first, int count, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  if (first < 0 || count < 0 || first + count > p->n_local) return fail(SRM_ERR_CONFIG, "subject range");
  if (count == 0) return SRM_OK;
  return run_stages(finalize_stages(p, first, count), as_stream(stream));
}

int srm_profile_finalize(srm_plan* p, float* ms_out, int capacity, int* n_out, void* stream) {
  if (!p || !p->ws || !ms_out || !n_out) return fail(SRM_ERR_CONFIG, "plan not bound");
  return profile_stages(finalize_stages(p, 0, p->n_local), ms_out, capacity, n_out, as_stream(stream));
}

int srm_prepare_gram_range(srm_plan* p, int first, int count, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  if (!(p->flags & SRM_FLAG_GRAM)) return SRM_OK;
  if (first < 0 || count < 0 || first + count > p->n_local) return fail(SRM_ERR_CONFIG, "subject range out of bounds");
  if (count == 0) return SRM_OK;
  for (int i = first; i < first + count; ++i) p->sliced[i] = 1;
  cudaStream_t st = as_stream(stream);
  // int8 Gram of more than one wave of tiles: batches of one wave, the
  // slicing of every batch on the side stream (17 KB CTAs that fit beside the
  // Gram's) and each batch's Gram, mirror and G slices on `st` after its slices
  const int per = p->ldx / 128 > 0 ? (int)(p->items_oz.size() / std::max(p->n_local, 1)) : 1;
  const int ctas = per + 2 * (int)(p->items_oz2.size() / std::max(p->n_local, 1));  // CTAs per subject
  const int batch = std::max(1, 148 / std::max(ctas, 1));
  static const bool batched = [] {  // SRM_B200_GRAM_BATCH=0: slice everything, then one Gram launch (test knob)
    const char* e = getenv("SRM_B200_GRAM_BATCH");
    return !(e && e[0] == '0');
  }();
  if ((p->flags & SRM_FLAG_GRAM_I8) && count > batch && batched) {
    const Lanes* ln = nullptr;
    int rc = plan_lanes(p, &ln);
    if (rc) return rc;
    const int nb = (count + batch - 1) / batch;
    while ((int)p->gram_events.size() < nb) {
      cudaEvent_t ev;
      const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "gram events");
      p->gram_events.push_back(ev);
    }
    while (!p->items_oz2.empty() && (int)p->pair_events.size() < nb) {
      cudaEvent_t ev;
      const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "gram events");
      p->pair_events.push_back(ev);
    }
    // the Gram batches run on a high-priority stream, so their CTAs are
    // dispatched ahead of pending slicing CTAs as SMs free up
    if (!p->hi_stream) {
      int lo = 0, hi = 0;
      cudaError_t e0 = cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (e0 == cudaSuccess) e0 = cudaStreamCreateWithPriority(&p->hi_stream, cudaStreamNonBlocking, hi);
      if (e0 == cudaSuccess) e0 = cudaStreamCreateWithPriority(&p->hi_stream2, cudaStreamNonBlocking, hi);
      if (e0 != cudaSuccess) return cuda_fail(e0, "gram stream");
    }
    // a batch's mirror and G row slices run on the second high-priority stream
    // behind the batch's Gram, so the next batch's Gram starts at once
    while ((int)p->post_events.size() < nb) {
      cudaEvent_t ev;
      const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "gram events");
      p->post_events.push_back(ev);
    }
    cudaStream_t gs = p->hi_stream, ps = p->hi_stream2;
    cudaError_t e = cudaEventRecord(ln->fork[1], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ln->side[1], ln->fork[1], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(gs, ln->fork[1], 0);
    for (int b = 0; b < nb && e == cudaSuccess; ++b) {
      const int f = first + b * batch, n = std::min(batch, first + count - f);
      e = gram_stages(p, f, n)[0].fn(ln->side[1]);  // oz_split
      if (e == cudaSuccess) e = cudaEventRecord(p->gram_events[b], ln->side[1]);
    }
    for (int b = 0; b < nb && e == cudaSuccess; ++b) {
      const int f = first + b * batch, n = std::min(batch, first + count - f);
      e = cudaStreamWaitEvent(gs, p->gram_events[b], 0);
      const std::vector<Stage> v = gram_stages(p, f, n);
      for (size_t k = 1; k < v.size() && e == cudaSuccess; ++k) {
        if (!strcmp(v[k].name, "oz_gram_pairs")) {
          // the pairs on a second high-priority stream, beside the batch's
          // single tiles: together one wave, as the single-CTA batch is
          e = cudaStreamWaitEvent(p->hi_stream2, p->gram_events[b], 0);
          if (e == cudaSuccess) e = v[k].fn(p->hi_stream2);
          if (e == cudaSuccess) e = cudaEventRecord(p->pair_events[b], p->hi_stream2);
          continue;
        }
        if (!strcmp(v[k].name, "oz_gram")) {
          e = v[k].fn(gs);
          if (e == cudaSuccess && !p->items_oz2.empty()) e = cudaStreamWaitEvent(gs, p->pair_events[b], 0);
          if (e == cudaSuccess) e = cudaEventRecord(p->post_events[b], gs);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(ps, p->post_events[b], 0);
          continue;
        }
        e = v[k].fn(ps);  // mirror_gram, oz_slice_g
      }
    }
    if (e == cudaSuccess) e = cudaEventRecord(ln->join[1], gs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ln->join[1], 0);
    if (e == cudaSuccess) e = cudaEventRecord(ln->join[2], ps);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ln->join[2], 0);
    return check(e, "prepare_gram");
  }
  for (const Stage& s : gram_stages(p, first, count)) {
    const cudaError_t e = s.fn(st);
    if (e != cudaSuccess) return cuda_fail(e, s.name);
  }
  return SRM_OK;
}

int srm_profile_gram(srm_plan* p, float* ms_out, int capacity, int* n_out, void* stream) {
  if (!p || !p->ws || !ms_out || !n_out) return fail(SRM_ERR_CONFIG, "plan not bound");
  if (!(p->flags & SRM_FLAG_GRAM)) {
    *n_out = 0;
    return SRM_OK;
  }
  return profile_stages(gram_stages(p, 0, p->n_local), ms_out, capacity, n_out, as_stream(stream));
}

int srm_prepare_gram(srm_plan* p, void* stream) {
  if (!p) return fail(SRM_ERR_CONFIG, "null plan");
  return srm_prepare_gram_range(p, 0, p->n_local, stream);
}

int srm_reset(srm_plan* p, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  return check(launch_reset(p->dp, as_stream(stream)), "reset");
}

int srm_read_status(srm_plan* p, int32_t* out4) {
  if (!p || !p->ws || !out4) return fail(SRM_ERR_CONFIG, "plan not bound");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "synchronize");
  e = cudaMemcpy(out4, p->dp.status, 16, cudaMemcpyDeviceToHost);
  return check(e, "read_status");
}

int srm_clear_status(srm_plan* p, void* stream) {
  if (!p || !p->ws) return fail(SRM_ERR_CONFIG, "plan not bound");
  return check(cudaMemsetAsync(p->dp.status, 0, 16, as_stream(stream)), "clear_status");
}

}  // extern "C"

// sg_plan.cu -- the launch planner: for every compiled M4RM variant and work split, an estimate
// from measured per-k-block / per-CTA costs (g_calib) or the analytic ALU / shared-memory model,
// and the cheapest plan; plus the streamed-B group order (streamed_order) of a product.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <tuple>
#include <vector>

#include <cudaTypedefs.h>

#include "sg_api_internal.h"

namespace sg {
namespace api {

struct Calib {
  int field, rt, threads, sched;
  double blk, cta;
};
const Calib g_calib[] = {
    {1, 1, 256, 0, 1008, 4776},  // max err 32%, 16 runs
    {1, 1, 256, 1, 1358, 9249},  // max err 8%, 16 runs
    {1, 2, 256, 0, 1246, 13806},  // max err 23%, 16 runs
    {1, 2, 256, 1, 1461, 15548},  // max err 5%, 16 runs
    {1, 2, 512, 0, 1937, 20379},  // max err 3%, 16 runs
    {1, 2, 512, 1, 1757, 23095},  // max err 5%, 16 runs
    {1, 4, 256, 0, 1498, 20872},  // max err 19%, 16 runs
    {1, 4, 256, 1, 1778, 22034},  // max err 4%, 16 runs
    {1, 4, 512, 0, 2531, 22821},  // max err 3%, 16 runs
    {1, 4, 512, 1, 2520, 23839},  // max err 1%, 16 runs
    {1, 8, 256, 0, 2435, 22269},  // max err 3%, 16 runs
    {1, 8, 256, 1, 2311, 23809},  // max err 2%, 16 runs
    {1, 8, 256, 2, 2332, 23947},  // max err 2%, 16 runs
    {1, 8, 512, 0, 3731, 22100},  // max err 2%, 17 runs
    {1, 8, 512, 1, 3909, 23979},  // max err 9%, 17 runs
    {1, 16, 256, 0, 3620, 21271},  // max err 2%, 17 runs
    {1, 16, 256, 1, 3690, 21923},  // max err 1%, 17 runs
    {1, 16, 256, 2, 3085, 22701},  // max err 3%, 17 runs
    {2, 1, 256, 0, 1751, 2566},  // max err 12%, 12 runs
    {2, 1, 256, 1, 2323, 4983},  // max err 2%, 11 runs
    {2, 2, 256, 0, 2224, 0},  // max err 20%, 12 runs
    {2, 2, 256, 1, 2597, 8949},  // max err 1%, 12 runs
    {2, 2, 512, 0, 3905, 13200},  // max err 1%, 12 runs
    {2, 2, 512, 1, 3491, 16819},  // max err 3%, 12 runs
    {2, 4, 256, 0, 3611, 11742},  // max err 2%, 12 runs
    {2, 4, 256, 1, 3230, 14751},  // max err 2%, 12 runs
    {2, 4, 256, 2, 3052, 14398},  // max err 3%, 12 runs
    {2, 4, 512, 0, 5787, 23269},  // max err 3%, 12 runs
    {2, 4, 512, 1, 5496, 29464},  // max err 6%, 12 runs
    {2, 8, 256, 0, 5078, 24707},  // max err 1%, 12 runs
    {2, 8, 256, 1, 4624, 27467},  // max err 3%, 12 runs
    {2, 8, 256, 2, 4280, 27483},  // max err 2%, 12 runs
    {3, 1, 256, 0, 1661, 6451},  // max err 8%, 10 runs
    {3, 1, 256, 1, 2286, 4824},  // max err 0%, 10 runs
    {3, 2, 256, 0, 2009, 6708},  // max err 11%, 11 runs
    {3, 2, 256, 1, 2522, 8210},  // max err 0%, 10 runs
    {3, 2, 512, 0, 3601, 12463},  // max err 1%, 11 runs
    {3, 2, 512, 1, 3372, 15226},  // max err 1%, 11 runs
    {3, 4, 256, 0, 3385, 11532},  // max err 2%, 11 runs
    {3, 4, 256, 1, 3121, 14450},  // max err 1%, 11 runs
    {3, 4, 256, 2, 2877, 12478},  // max err 5%, 11 runs
    {3, 4, 512, 0, 5032, 24646},  // max err 1%, 11 runs
    {3, 4, 512, 1, 4885, 29181},  // max err 2%, 11 runs
    {3, 8, 256, 0, 4661, 24285},  // max err 1%, 11 runs
    {3, 8, 256, 1, 4440, 27624},  // max err 1%, 11 runs
    {3, 8, 256, 2, 3870, 27697},  // max err 1%, 11 runs
    {4, 1, 256, 0, 891, 9118},  // max err 13%, 10 runs
    {4, 1, 256, 1, 1296, 3985},  // max err 0%, 10 runs
    {4, 2, 256, 0, 1154, 5752},  // max err 9%, 11 runs
    {4, 2, 256, 1, 1419, 5412},  // max err 0%, 10 runs
    {4, 2, 512, 0, 1844, 7143},  // max err 1%, 11 runs
    {4, 2, 512, 1, 1750, 7672},  // max err 6%, 11 runs
    {4, 4, 256, 0, 1817, 7237},  // max err 1%, 11 runs
    {4, 4, 256, 1, 1738, 7639},  // max err 3%, 11 runs
    {4, 4, 512, 0, 2540, 14624},  // max err 0%, 12 runs
    {4, 4, 512, 1, 2446, 15162},  // max err 1%, 12 runs
    {4, 8, 256, 0, 2398, 13635},  // max err 1%, 12 runs
    {4, 8, 256, 1, 2302, 14121},  // max err 2%, 12 runs
    {4, 8, 256, 2, 2324, 10497},  // max err 7%, 12 runs
    {4, 8, 512, 0, 3690, 26807},  // max err 2%, 12 runs
    {4, 8, 512, 1, 3643, 27070},  // max err 1%, 12 runs
    {4, 16, 256, 0, 3598, 26686},  // max err 1%, 12 runs
    {4, 16, 256, 1, 3547, 27403},  // max err 2%, 12 runs
    {4, 16, 256, 2, 3107, 27836},  // max err 3%, 12 runs
    // GF(4) RT 16 with 8 builder warps (schedule 5): the schedule-2 constants x 0.978, its measured
    // ratio on 8192^3 (tools/step_probe.py, profiles/r02y_step_gf4.txt: 1.312 -> 1.283 ms)
    {4, 16, 256, 5, 3038, 27836},
    // F3 with the second accumulator set in TMEM (schedule 6, 8192 rows per CTA): from the
    // bench-style steps of 32768^3 split-K (76.8 ms) and 8192 x 32768^2 stream-K (19.5 ms)
    // (tools/step_probe.py, profiles/r02af_step.txt, r02ag_step.txt)
    {1, 32, 256, 6, 5300, 25000},
    // GF(4), schedule 6: 8192^3 stream-K 1.036 ms (profiles/r02ah_step.txt)
    {4, 32, 256, 6, 4370, 25000},
    // F7, schedule 6 (4096 rows per CTA): 16384 x 8192 x 16384 stream-K 12.55 ms (r02aj_step.txt)
    {3, 16, 256, 6, 6930, 25000},
    // F5, schedule 6 (4096 rows per CTA, row-slots rotating through three TMEM regions):
    // 8192^3 stream-K 3.468 ms, 4096^3 0.470 ms (profiles/r02ba_step.txt)
    {2, 16, 256, 6, 7550, 25000},
    // fused one-launch variants (schedule + 10), from bench-style step times on small shapes
    // (tools/step_probe.py --grid, profiles/r02n_step_grid.jsonl; fit: tools/fit_calib.py)
    {1, 1, 256, 10, 1329, 0},  // max err 36%, 20 runs
    {1, 2, 256, 10, 1666, 2563},  // max err 16%, 19 runs
    {1, 2, 256, 11, 1661, 4742},  // max err 10%, 14 runs
    {1, 4, 256, 10, 2051, 4472},  // max err 19%, 19 runs
    {1, 4, 256, 11, 2264, 6335},  // max err 19%, 16 runs
    {2, 1, 256, 10, 2492, 2328},  // max err 14%, 17 runs
    {2, 2, 256, 10, 3004, 5534},  // max err 18%, 20 runs
    {2, 2, 256, 11, 3011, 6862},  // max err 9%, 14 runs
    {2, 4, 256, 10, 3893, 7254},  // max err 12%, 16 runs
    {2, 4, 256, 11, 3797, 8881},  // max err 20%, 16 runs
    {3, 1, 256, 10, 2466, 1696},  // max err 12%, 17 runs
    {3, 2, 256, 10, 3033, 5415},  // max err 19%, 20 runs
    {3, 2, 256, 11, 3054, 6702},  // max err 9%, 14 runs
    {3, 4, 256, 10, 3729, 7411},  // max err 11%, 16 runs
    {3, 4, 256, 11, 3778, 9369},  // max err 19%, 16 runs
    {4, 1, 256, 10, 1682, 2093},  // max err 9%, 17 runs
    {4, 2, 256, 10, 1886, 2951},  // max err 14%, 19 runs
    {4, 2, 256, 11, 1903, 5482},  // max err 9%, 14 runs
    {4, 4, 256, 10, 2248, 4848},  // max err 12%, 16 runs
    {4, 4, 256, 11, 2386, 7073},  // max err 18%, 17 runs
};

// experiments: SG_STREAMK_HYBRID=0 plans pure stream-K ranges (no whole-tile waves)
static const bool g_streamk_hybrid = [] {
  const char* e = getenv("SG_STREAMK_HYBRID");
  return !e || atoi(e) != 0;
}();

const Calib* calib_for(const KernelInfo* ki) {
  if (ki->k != 8) return nullptr;
  const int sched = ki->sched + (ki->fn_fused ? SCHED_FUSED : 0);
  for (const Calib& c : g_calib)
    if (c.field == ki->field && c.rt == ki->rt && c.threads == ki->threads && c.sched == sched) return &c;
  if (ki->fn_fused)  // uncalibrated fused variant: its unfused twin's constants
    for (const Calib& c : g_calib)
      if (c.field == ki->field && c.rt == ki->rt && c.threads == ki->threads && c.sched == ki->sched) return &c;
  return nullptr;
}

// Per-lane (4 words) ALU instructions and shared-memory bytes per (row, k-block), and the
// table-build ALU work per entry; see DESIGN.md "Planner".
void field_costs(int f, double* lane_alu, double* lane_smem, double* entry_alu) {
  switch (f) {
    case SG_F2: *lane_alu = 4 + 3; *lane_smem = 16 + 4; *entry_alu = 4 + 8; break;
    case SG_F3: *lane_alu = 36 + 6; *lane_smem = 64 + 8; *entry_alu = 20 + 16; break;
    case SG_GF4: *lane_alu = 12 + 6; *lane_smem = 64 + 8; *entry_alu = 8 + 16; break;
    case SG_F5: *lane_alu = 80 + 9; *lane_smem = 144 + 12; *entry_alu = 48 + 24; break;
    case SG_GF8: *lane_alu = 28 + 9; *lane_smem = 144 + 12; *entry_alu = 12 + 24; break;
    case SG_Z4: *lane_alu = 12 + 6; *lane_smem = 64 + 8; *entry_alu = 12 + 16; break;
    case SG_Z8: *lane_alu = 36 + 9; *lane_smem = 144 + 12; *entry_alu = 28 + 24; break;
    default: *lane_alu = 72 + 9; *lane_smem = 144 + 12; *entry_alu = 40 + 24; break;
  }
}

int make_plan_uncached(int field, int64_t m, int64_t l, int64_t n, int k, int device, Plan* out);

// Plans are pure functions of the shape, the device and the overrides: cache them so repeated
// products (the common case) skip the search (callers hold g_mu).
int make_plan(int field, int64_t m, int64_t l, int64_t n, int k, int device, Plan* out) {
  typedef std::tuple<int, int64_t, int64_t, int64_t, int, int, int, int, int, int, int, int> Key;
  static std::map<Key, Plan> cache;
  const Key key{field, m, l, n, std::min(k, 8), device, g_override_rt, g_override_splits, g_override_pipe,
                g_override_threads, g_ablation, g_sm_reserve};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return SG_OK;
  }
  const int rc = make_plan_uncached(field, m, l, n, k, device, out);
  if (rc == SG_OK) {
    if (cache.size() > 4096) cache.clear();
    cache[key] = *out;
  }
  return rc;
}

int make_plan_uncached(int field, int64_t m, int64_t l, int64_t n, int k, int device, Plan* out) {
  DevState& ds0 = dev_state(device);
  DevState ds = ds0;
  ds.sms = std::max(1, ds0.sms - g_sm_reserve);  // CTAs for sms - reserve SMs: the rest stay free
  const int K = std::min(k, 8);
  const int64_t wc32 = 2 * w64_of(n), wa32 = 2 * w64_of(l);
  const int nblocks = (int)((l + K - 1) / K);
  const int64_t slabs = (wc32 + SLAB_WORDS - 1) / SLAB_WORDS;
  double lane_alu, lane_smem, entry_alu;
  field_costs(field, &lane_alu, &lane_smem, &entry_alu);
  const int R = planes(field);
  const bool small0 = K == 8 && (double)m * (double)l * (double)n <= 2.0e9;
  Plan best;
  best.est_clk = 1e300;
  // pass 0: fused plans for small products only; pass 1 (no plan fits, e.g. > 65535 row groups):
  // every variant
  for (int pass = 0; pass < 2 && !best.ki; ++pass)
  for (int i = 0; i < m4rm_kernel_count(); ++i) {
    // (pass 1: `small` equals the variant's own kind, so the size filter below keeps everything)
    const bool small = pass == 0 ? small0 : m4rm_kernel_at(i)->fn_fused != nullptr;
    KernelInfo* ki = m4rm_kernel_at(i);
    if (ki->field != field || ki->k != K) continue;
    if (g_override_rt && ki->rt != g_override_rt) continue;
    const bool fused = ki->fn_fused != nullptr;
    if (g_override_pipe >= 0 && ki->sched + (fused ? SCHED_FUSED : 0) != g_override_pipe) continue;
    // Products up to ~2e9 mul-adds run the fused one-launch kernel, larger ones the unfused
    // variants (bench-style steps, profiles/r02n_step_grid.jsonl: the best fused plan beat the best
    // unfused one on every shape up to 1.07e9 mul-adds, by 10-40 %, and lost on every shape from
    // 4.3e9 up).  A forced schedule (sg_set_plan_override) overrides the split.
    if (g_override_pipe < 0 && fused != small) continue;
    if (g_override_threads && ki->threads != g_override_threads) continue;
    if (ki->ablation != g_ablation) continue;
    if (ki->occupancy < 1) continue;  // does not fit this device
    const int rows = ki->rt * ki->threads;
    const int64_t rgroups = (m + rows - 1) / rows;
    const double E = (double)(1 << K);
    const double alu_l = rows * lane_alu / 64.0, alu_t = E * entry_alu / 64.0;
    const double smem_l = (rows * lane_smem + rows * R * 4.0) / 128.0, smem_t = E * R * ENTRY_BYTES / 128.0;
    // serial: table build then lookups; pipelined / warp-specialized: both share the pipes
    const double t_block = ws_tma(ki->sched) ? std::max(alu_l + alu_t, smem_l + smem_t) + 100.0
                           : ki->sched == 1 ? std::max(alu_l + alu_t, smem_l + smem_t) + 250.0
                                            : std::max(alu_l, smem_l) + std::max(alu_t, smem_t) + 400.0;
    const Calib* cal = calib_for(ki);
    const int occ = std::max(1, ki->occupancy);
    const int max_splits = std::max(1, std::min(nblocks, 64));
    const int64_t tiles = slabs * rgroups;
    const int64_t units = tiles * nblocks;
    if (!fused) {
      // stream-K candidate: one wave of SMs x occupancy CTAs, each owning U / G consecutive
      // (tile, k-block) units, then a compact reduction of the partially covered tiles
      const int64_t G = (int64_t)ds.sms * occ;
      // Hybrid: with at least one tile per CTA the leading tiles/G whole waves go tile by tile
      // (CTA c: tiles c, c + G, ...), all CTAs walking the k-blocks of neighbouring tiles together,
      // and only the last, partial wave is cut into unit ranges -- pure stream-K ranges of several
      // tiles scatter the concurrent CTAs over all of k and the row groups, and B and A's index
      // words then stream from HBM for every tile (F3 32768^3: 72 GB per launch against 2 GB).
      const int64_t dp = g_streamk_hybrid && G > 0 && tiles >= G ? tiles / G * G : 0;
      const int64_t units_sk = (tiles - dp) * nblocks;
      // a CTA's range: partial tail, whole tiles, partial head (one segment boundary each).  Ranges
      // of more than ~2 tiles (no hybrid: fewer tiles than CTAs never have them) are planned only
      // when A's index words and B fit in L2 together; forced plans (splits = -1) take any range.
      const int rpw = field == SG_F2 ? 4 : planes(field) == 3 ? 1 : 2;
      const double l2_set = (double)((nblocks + rpw - 1) / rpw) * rgroups * rows * 4.0 + (double)R * l * wc32 * 4.0;
      const bool short_ranges = G > 0 && (units_sk + G - 1) / G <= 2 * (int64_t)nblocks - 1;
      const bool ok = K == 8 && (g_override_splits == 0 || g_override_splits == -1) && G > 0 && units >= G &&
                      (short_ranges || l2_set <= 120e6 || g_override_splits == -1 || (ki->sched == 6 && rgroups <= 4));
      if (ok) {
        const double per = (double)(units + G - 1) / G, per_sk = (double)(units_sk + G - 1) / G;
        // segments per CTA: its whole tiles, then the ends of its unit range
        const double nseg = (double)(dp / G) + (units_sk ? std::min(2.0, per_sk) + std::floor(per_sk / nblocks) : 0.0);
        const double t_cta = cal ? per * cal->blk + nseg * cal->cta : 1.25 * (per * t_block + 3000.0 * nseg);
        const double bytes = (double)G * 2.0 * R * rows * 16.0 + (double)R * m * wc32 * 4.0;
        // occ co-resident CTAs share the SM, as in the split-K estimate below
        const double est = occ * t_cta + bytes / 3000.0 + 8000.0;
        if (est < best.est_clk) {
          best.est_clk = est;
          best.ki = ki;
          best.kernel_index = i;
          best.splits = 1;
          best.bps = nblocks;
          best.mpad = rgroups * rows;
          best.streamk = true;
          best.units = units_sk;
          best.dp_tiles = dp;
          best.tiles = tiles;
          best.slabs = (int)slabs;
          best.rows = rows;
          best.grid = dim3((unsigned)G, 1, 1);
        }
      }
    }
    for (int sp = 1; sp <= max_splits; ++sp) {
      if (g_override_splits && sp != g_override_splits) continue;
      const int bps = (nblocks + sp - 1) / sp;
      const int splits = (nblocks + bps - 1) / bps;
      if (splits != sp) continue;
      if (rgroups > 65535 || splits > 65535) continue;  // grid.y / grid.z limits (stream-K has none)
      const double ctas = (double)slabs * rgroups * splits;
      // a fused plan's split-K CTAs meet in the kernel: all of them co-resident (one wave)
      if (fused && splits > 1 && ctas > (double)ds.sms * occ) continue;
      // calibrated variants: measured per-block and per-CTA clocks; others: the analytic
      // model with a 25 % penalty, so a measured variant wins unless clearly worse
      // (fused variants use their unfused twin's calibration)
      const double t_cta = cal ? bps * cal->blk + cal->cta : 1.25 * (bps * t_block + 3000.0);
      const double waves = std::ceil(ctas / (ds.sms * occ));
      double est = waves * t_cta * std::min<double>(occ, ctas / ds.sms > 1 ? occ : 1);
      if (splits > 1) {
        const double bytes = (splits + 1.0) * R * (double)m * wc32 * 4.0;
        // ~3 KB/clk HBM + one extra launch (fused: the meeting inside the kernel instead)
        est += bytes / 3000.0 + (fused ? 1500.0 : 8000.0);
      }
      if (fused) est -= 6000.0;  // no index pre-pass launch
      if (est < best.est_clk) {
        best.est_clk = est;
        best.ki = ki;
        best.kernel_index = i;
        best.splits = splits;
        best.bps = bps;
        best.mpad = rgroups * rows;
        best.streamk = false;
        best.dp_tiles = 0;
        best.grid = dim3((unsigned)slabs, (unsigned)rgroups, (unsigned)splits);
      }
    }
  }
  if (!best.ki)
    return fail(SG_EUNSUPPORTED, "no compiled M4RM kernel matches the request (check sg_set_plan_override; more "
                                 "than 65535 row groups need the k = 8 stream-K plan)");
  best.K = K;
  best.nblocks = nblocks;
  best.wa32 = (int)wa32;
  best.wc32 = (int)wc32;
  if (best.ki->fn_fused) {  // A's words are staged by the kernel itself
    best.at_words = 0;
    best.at_planes = 0;
  } else if (K == 8) {
    const int rpw = field == SG_F2 ? 4 : planes(field) == 3 ? 1 : 2;
    best.at_words = (nblocks + rpw - 1) / rpw;
    best.at_planes = 1;
  } else {
    best.at_words = (int)wa32;
    best.at_planes = R;
  }
  if (best.grid.y > 65535) return fail(SG_EUNSUPPORTED, "too many row groups for one launch");
  *out = best;
  return SG_OK;
}

// B's planes as a 3-D u32 tensor {words, rows, planes} with a {4, 8, R} box: one TMA copy stages
// one k-block of a 128-column slab (rows past l and words past wc32 arrive as zeros).
bool encode_b_map(CUtensorMap* map, const void* B, int field, int64_t l, int wc32) {
  static PFN_cuTensorMapEncodeTiled encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }();
  if (!encode || l <= 0) return false;
  const cuuint32_t R = (cuuint32_t)planes(field);
  const cuuint64_t dims[3] = {(cuuint64_t)wc32, (cuuint64_t)l, R};
  const cuuint64_t strides[2] = {(cuuint64_t)wc32 * 4, (cuuint64_t)l * wc32 * 4};
  const cuuint32_t box[3] = {4, 8, R};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(B), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t workspace_bytes_for(const Plan& p, int field) {
  const int R = planes(field);
  int64_t b = (int64_t)p.at_planes * p.at_words * p.mpad * 4;
  b = (b + 255) / 256 * 256;
  if (p.streamk) b += (int64_t)p.grid.x * SK_SLOTS * R * p.rows * SLAB_WORDS * 4;
  else if (p.splits > 1 && p.ki->fn_fused)  // compact slots [split][tile][R][rows][4 words]
    b += (int64_t)p.splits * R * p.mpad * ((p.wc32 + SLAB_WORDS - 1) / SLAB_WORDS) * SLAB_WORDS * 4;
  else if (p.splits > 1) b += (int64_t)p.splits * R * p.mpad * p.wc32 * 4;
  return std::max<int64_t>(b, 256);
}


// One stream-K wave of the warp-specialized kernel: its builder warps stage every k-block by
// TMA, so they can wait for each block's chunk; the 4-block group order needs nblocks % 4 == 0.
bool streamable(const Plan& p) {
  return p.streamk && p.dp_tiles == 0 && ws_tma(p.ki->sched) && p.ki->fn_stream && p.K == 8 && p.wc32 % 4 == 0 && p.nblocks % 4 == 0 &&
         p.tiles > 0 && p.nblocks / 4 <= STRM_MAX_GROUPS && (int64_t)p.tiles * (p.nblocks / 4) <= (int64_t)1 << 24;
}

typedef std::tuple<int, int, int64_t, int64_t, int64_t, unsigned> PermKey;
std::map<PermKey, int*> g_perm;  // device copies of streamed_order, per (device, plan)
PermKey perm_key(const Plan& p, int dev, int64_t m, int64_t l, int64_t n) {
  return PermKey{dev, p.kernel_index, m, l, n, p.grid.x};
}

// Per tile, the order in which a streamed product consumes B's 4-block groups.  Each group gets
// the earliest time (k-blocks into its CTA's range) at which one of the tile's stream-K segments
// needs it, and groups are numbered in that order: B goes up in k order, so every CTA starts on
// blocks that arrive first, and a tile's contributors share the arrivals instead of some CTAs
// waiting for blocks deep in k.  virtual group v of tile t -> real group perm[t * ng + v].
std::vector<int> streamed_order(const Plan& p) {
  const int nb = p.nblocks, ng = nb / 4;
  const int64_t U = p.units, G = p.grid.x;
  std::vector<int> perm((size_t)p.tiles * ng);
  std::vector<std::pair<int64_t, int>> need(ng);
  for (int64_t t = 0; t < p.tiles; ++t) {
    for (int g = 0; g < ng; ++g) need[g] = {INT64_MAX, g};
    const int64_t lo = t * nb, hi = lo + nb;
    int64_t c = lo * G / U;
    while (c > 0 && c * U / G > lo) --c;
    while ((c + 1) * U / G <= lo) ++c;
    for (; c < G && c * U / G < hi; ++c) {
      const int64_t u0 = c * U / G, u1 = (c + 1) * U / G;
      const int64_t a = std::max(u0, lo), b = std::min(u1, hi);
      for (int64_t g = (a - lo) / 4; a < b && g <= (b - 1 - lo) / 4; ++g) {
        const int64_t first = std::max(a, lo + 4 * g);  // the segment's first block in group g
        need[g].first = std::min(need[g].first, first - u0);
      }
    }
    std::sort(need.begin(), need.end());  // by (time, group)
    for (int i = 0; i < ng; ++i) perm[t * ng + need[i].second] = i;
  }
  return perm;
}

// Plan a streamed product and upload its group order (callers hold g_mu).  Returns SG_OK, or
// SG_EUNSUPPORTED when the product cannot stream (the caller then uploads B first).
int prepare_streamed(int field, int64_t m, int64_t l, int64_t n, int k, int dev, Plan* out) {
  int rc = make_plan(field, m, l, n, k, dev, out);
  if (rc != SG_OK) return rc;
  if (!streamable(*out)) return SG_EUNSUPPORTED;
  const PermKey key = perm_key(*out, dev, m, l, n);
  if (g_perm.count(key)) return SG_OK;
  const std::vector<int> perm = streamed_order(*out);
  int* d = nullptr;
  SG_CUDA(cudaMalloc(&d, perm.size() * sizeof(int)), "streamed order alloc");
  SG_CUDA(cudaMemcpy(d, perm.data(), perm.size() * sizeof(int), cudaMemcpyHostToDevice), "streamed order upload");
  if (g_perm.size() > 256) g_perm.clear();  // (leaks the old device arrays; bounded by the cap)
  g_perm[key] = d;
  return SG_OK;
}

const int* streamed_order_on_device(const Plan& p, int dev, int64_t m, int64_t l, int64_t n) {
  auto it = g_perm.find(perm_key(p, dev, m, l, n));
  return it == g_perm.end() ? nullptr : it->second;
}

}  // namespace api
}  // namespace sg

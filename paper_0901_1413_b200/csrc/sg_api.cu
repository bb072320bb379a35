// sg_api.cu -- the C ABI (include/slicegemm_b200.h): argument checks, the launch planner,
// workspace management, the host-buffer entry point, timing and launch accounting.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>

#include <cudaTypedefs.h>

#include "../../include/slicegemm_b200.h"
#include "sg_field.cuh"
#include "sg_internal.h"

using namespace sg;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_streamed{0};  // host-buffer products that streamed B (sg_host_streamed_count)
int g_override_rt = 0, g_override_splits = 0, g_override_pipe = -1, g_override_threads = 0, g_ablation = 0;
int g_sm_reserve = 0;  // SMs the planner leaves free (for a collective running concurrently)
bool g_timing = false;
double g_last_ms[3] = {0, 0, 0};
std::mutex g_mu;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(SG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define SG_CUDA(call, where)                        \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

bool valid_field(int f) { return f >= SG_F2 && f <= SG_Z8; }
int planes(int f) { return f == SG_F2 ? 1 : (f == SG_F5 || f == SG_F7 || f == SG_GF8 || f == SG_Z8) ? 3 : 2; }
int64_t w64_of(int64_t n) { return (n + 63) / 64; }

// ---------------------------------------------------------------- per-device state
struct DevState {
  bool attrs_set = false;
  int sms = 148;
};
std::map<int, DevState> g_dev;

DevState& dev_state(int device) {
  DevState& d = g_dev[device];
  if (!d.attrs_set) {
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device);
    for (int i = 0; i < m4rm_kernel_count(); ++i) {
      KernelInfo* k = m4rm_kernel_at(i);
      cudaFuncSetAttribute(k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem_bytes);
      if (k->fn_stream &&
          cudaFuncSetAttribute(k->fn_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem_stream) != cudaSuccess)
        k->fn_stream = nullptr;  // does not fit this device: no streamed variant
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, k->fn) == cudaSuccess) k->regs = fa.numRegs;
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k->fn, k->launch_threads, k->smem_bytes);
      k->occupancy = occ;
    }
    cudaGetLastError();
    d.attrs_set = true;
  }
  return d;
}

// Workspace cache keyed by (device, stream): stream-ordered reuse is safe, cross-stream is not.
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};
std::map<std::pair<int, cudaStream_t>, Buf> g_ws;
std::map<int, int*> g_flags;  // per-device error flag for pack / unpack

int* flag_for(int device, cudaError_t* err) {
  int*& f = g_flags[device];
  *err = cudaSuccess;
  if (!f) *err = cudaMalloc(&f, 16);
  return *err == cudaSuccess ? f : nullptr;
}

void* workspace_for(int device, cudaStream_t st, size_t bytes, cudaError_t* err) {
  Buf& b = g_ws[{device, st}];
  *err = cudaSuccess;
  if (b.bytes < bytes) {
    if (b.p) {
      cudaStreamSynchronize(st);
      cudaFree(b.p);
    }
    b.p = nullptr;
    b.bytes = 0;
    *err = cudaMalloc(&b.p, bytes);
    if (*err != cudaSuccess) return nullptr;
    b.bytes = bytes;
  }
  return b.p;
}

// ---------------------------------------------------------------- planner
struct Plan {
  KernelInfo* ki = nullptr;
  int kernel_index = -1;
  int K = 8, splits = 1, bps = 0, nblocks = 0;
  int64_t mpad = 0;
  int wa32 = 0, wc32 = 0;
  int at_words = 0, at_planes = 0;  // staged index array: k=8 packed words (1 plane), else A^T planes
  bool streamk = false;              // one wave of CTAs over tiles x k-blocks (see m4rm_kernel)
  int64_t units = 0, tiles = 0;
  int slabs = 0, rows = 0;
  dim3 grid;
  double est_clk = 0;
};

// Measured per-CTA cost of the k = 8 variants on B200 (tools/tune.py over BASELINE.json's configs
// and the per-rank shapes of the sharded runs, fitted by tools/fit_calib.py to the model below;
// profiles/r01d_tune_all.jsonl): {field, rows per thread, lookup threads, schedule, clocks per
// k-block, clocks per CTA}.
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
};

const Calib* calib_for(const KernelInfo* ki) {
  if (ki->k != 8) return nullptr;
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
  Plan best;
  best.est_clk = 1e300;
  for (int i = 0; i < m4rm_kernel_count(); ++i) {
    KernelInfo* ki = m4rm_kernel_at(i);
    if (ki->field != field || ki->k != K) continue;
    if (g_override_rt && ki->rt != g_override_rt) continue;
    if (g_override_pipe >= 0 && ki->sched != g_override_pipe) continue;
    if (g_override_threads && ki->threads != g_override_threads) continue;
    if (ki->ablation != g_ablation) continue;
    if (ki->occupancy < 1) continue;  // does not fit this device
    const int rows = ki->rt * ki->threads;
    const int64_t rgroups = (m + rows - 1) / rows;
    const double E = (double)(1 << K);
    const double alu_l = rows * lane_alu / 64.0, alu_t = E * entry_alu / 64.0;
    const double smem_l = (rows * lane_smem + rows * R * 4.0) / 128.0, smem_t = E * R * ENTRY_BYTES / 128.0;
    // serial: table build then lookups; pipelined / warp-specialized: both share the pipes
    const double t_block = ki->sched == 2   ? std::max(alu_l + alu_t, smem_l + smem_t) + 100.0
                           : ki->sched == 1 ? std::max(alu_l + alu_t, smem_l + smem_t) + 250.0
                                            : std::max(alu_l, smem_l) + std::max(alu_t, smem_t) + 400.0;
    const Calib* cal = calib_for(ki);
    const int occ = std::max(1, ki->occupancy);
    const int max_splits = std::max(1, std::min(nblocks, 64));
    const int64_t tiles = slabs * rgroups;
    const int64_t units = tiles * nblocks;
    {
      // stream-K candidate: one wave of SMs x occupancy CTAs, each owning U / G consecutive
      // (tile, k-block) units, then a compact reduction of the partially covered tiles
      const int64_t G = (int64_t)ds.sms * occ;
      // a CTA's range: partial tail, whole tiles, partial head (one segment boundary each).  Ranges
      // of more than ~2 tiles scatter the concurrent CTAs over row groups, so they are planned only
      // when A's index words and B fit in L2 together (measured: F7 16384x8192x16384 -1.7 %,
      // F3 32768^3 +1.7 % where they do not); forced plans (splits = -1) take any range.
      const int rpw = field == SG_F2 ? 4 : planes(field) == 3 ? 1 : 2;
      const double l2_set = (double)((nblocks + rpw - 1) / rpw) * rgroups * rows * 4.0 + (double)R * l * wc32 * 4.0;
      const bool short_ranges = (units + G - 1) / G <= 2 * (int64_t)nblocks - 1;
      const bool ok = K == 8 && (g_override_splits == 0 || g_override_splits == -1) && G > 0 && units >= G &&
                      (short_ranges || l2_set <= 120e6 || g_override_splits == -1);
      if (ok) {
        const double per = (double)(units + G - 1) / G;
        const double nseg = std::min(2.0, per) + std::floor(per / nblocks);  // segments per CTA
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
          best.units = units;
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
      const double ctas = (double)slabs * rgroups * splits;
      // calibrated variants: measured per-block and per-CTA clocks; others: the analytic
      // model with a 25 % penalty, so a measured variant wins unless clearly worse
      const double t_cta = cal ? bps * cal->blk + cal->cta : 1.25 * (bps * t_block + 3000.0);
      const double waves = std::ceil(ctas / (ds.sms * occ));
      double est = waves * t_cta * std::min<double>(occ, ctas / ds.sms > 1 ? occ : 1);
      if (splits > 1) {
        const double bytes = (splits + 1.0) * R * (double)m * wc32 * 4.0;
        est += bytes / 3000.0 + 8000.0;  // ~3 KB/clk HBM + one extra launch
      }
      if (est < best.est_clk) {
        best.est_clk = est;
        best.ki = ki;
        best.kernel_index = i;
        best.splits = splits;
        best.bps = bps;
        best.mpad = rgroups * rows;
        best.streamk = false;
        best.grid = dim3((unsigned)slabs, (unsigned)rgroups, (unsigned)splits);
      }
    }
  }
  if (!best.ki) return fail(SG_EUNSUPPORTED, "no compiled M4RM kernel matches the request (check sg_set_plan_override)");
  best.K = K;
  best.nblocks = nblocks;
  best.wa32 = (int)wa32;
  best.wc32 = (int)wc32;
  if (K == 8) {
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
  else if (p.splits > 1) b += (int64_t)p.splits * R * p.mpad * p.wc32 * 4;
  return std::max<int64_t>(b, 256);
}

int check_mul_args(int field, const void* A, const void* B, const void* C, int64_t m, int64_t l,
                   int64_t n, int k) {
  if (!valid_field(field)) return fail(SG_EINVAL, "unknown field code");
  if (m < 0 || l < 0 || n < 0) return fail(SG_EINVAL, "negative dimension");
  if (k < 1 || k > 16) return fail(SG_EINVAL, "k must be in 1..16 (SPEC.md:306-311)");
  if (2 * w64_of(l) > 0x7fffffffLL || 2 * w64_of(n) > 0x7fffffffLL) return fail(SG_EINVAL, "dimension too large");
  if (m && n && (!C || (l && (!A || !B)))) return fail(SG_EINVAL, "null matrix pointer");
  if (m && n && l && A != (const void*)1) {  // (const void*)1: shape-only queries
    // the product reads A and B while it writes C
    const int R = planes(field);
    auto overlap = [](const void* p, int64_t pb, const void* q, int64_t qb) {
      const char* a = (const char*)p;
      const char* b = (const char*)q;
      return a < b + qb && b < a + pb;
    };
    const int64_t ab = (int64_t)R * m * w64_of(l) * 8, bb = (int64_t)R * l * w64_of(n) * 8,
                  cb = (int64_t)R * m * w64_of(n) * 8;
    if (overlap(C, cb, A, ab) || overlap(C, cb, B, bb)) return fail(SG_EINVAL, "C overlaps an operand");
  }
  return SG_OK;
}

// ---------------------------------------------------------------- streamed B (sg_m4rm_host)
// A product whose B arrives chunk by chunk while it runs (see M4rmArgs.ready).
struct StreamIn {
  const unsigned* ready;
  unsigned epoch;
  int first_groups;  // B's chunk j = 4-block groups [g0 (2^j - 1), g0 (2^(j+1) - 1)), g0 = first_groups
  int nchunks;
  unsigned* err;
};

// One stream-K wave of the warp-specialized kernel: its builder warps stage every k-block by
// TMA, so they can wait for each block's chunk; the 4-block group order needs nblocks % 4 == 0.
bool streamable(const Plan& p) {
  return p.streamk && p.ki->sched == 2 && p.ki->fn_stream && p.K == 8 && p.wc32 % 4 == 0 && p.nblocks % 4 == 0 &&
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

int m4rm_device(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l, int64_t n,
                int k, void* workspace, int64_t workspace_bytes, cudaStream_t stream, const StreamIn* sin);

}  // namespace

// ==================================================================== C ABI
extern "C" {

int sg_abi_version(void) { return SG_ABI_VERSION; }
const char* sg_last_error(void) { return g_err.c_str(); }
int sg_field_planes(int field) { return valid_field(field) ? planes(field) : -1; }
int64_t sg_launch_count(void) { return g_launches.load(); }
int64_t sg_host_streamed_count(void) { return g_streamed.load(); }

int sg_kernel_info(int index, int device, int* field, int* k, int* rows_per_thread, int* threads, int* schedule,
                   int* occupancy, int* regs, int* smem_bytes) {
  const int count = m4rm_kernel_count();
  if (index < 0 || index >= count) return -1;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lk(g_mu);
  dev_state(device);  // fills registers and occupancy
  const KernelInfo* ki = m4rm_kernel_at(index);
  if (field) *field = ki->field;
  if (k) *k = ki->k;
  if (rows_per_thread) *rows_per_thread = ki->rt;
  if (threads) *threads = ki->threads;
  if (schedule) *schedule = ki->sched;
  if (occupancy) *occupancy = ki->occupancy;
  if (regs) *regs = ki->regs;
  if (smem_bytes) *smem_bytes = ki->smem_bytes;
  cudaSetDevice(cur);
  return count;
}

int sg_set_plan_override(int rows_per_thread, int splits, int pipe, int threads) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_override_threads = threads;
  g_override_rt = rows_per_thread;
  g_override_splits = splits;
  g_override_pipe = pipe < 0 ? -1 : pipe;
  return SG_OK;
}

int sg_set_sm_reserve(int sms) {
  if (sms < 0 || sms > 64) return fail(SG_EINVAL, "SM reserve must be in 0..64");
  std::lock_guard<std::mutex> lk(g_mu);
  g_sm_reserve = sms;
  return SG_OK;
}

int sg_debug_ablation(int mask) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_ablation = mask;
  return SG_OK;
}

int sg_set_timing(int enable) {
  g_timing = enable != 0;
  return SG_OK;
}

int sg_last_timing(double* t, double* mm, double* r) {
  if (t) *t = g_last_ms[0];
  if (mm) *mm = g_last_ms[1];
  if (r) *r = g_last_ms[2];
  return SG_OK;
}

int sg_pack(int field, const uint8_t* dense, int64_t m, int64_t n, int64_t ld, uint64_t* planes_out,
            void* stream) {
  if (!valid_field(field)) return fail(SG_EINVAL, "unknown field code");
  if (m < 0 || n < 0 || ld < n) return fail(SG_EINVAL, "bad shape or leading dimension");
  if (m == 0 || n == 0) return SG_OK;
  if (!dense || !planes_out) return fail(SG_EINVAL, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e;
  int* flag = flag_for(dev, &e);
  if (!flag) return cuda_fail(e, "sg_pack flag");
  SG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st), "sg_pack");
  SG_CUDA(launch_pack(field, dense, m, n, ld, planes_out, flag, st), "sg_pack launch");
  g_launches++;
  int h = 0;
  SG_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "sg_pack");
  SG_CUDA(cudaStreamSynchronize(st), "sg_pack");
  if (h) return fail(SG_ERANGE, "entries out of range for the field");
  return SG_OK;
}

int sg_unpack(int field, const uint64_t* planes_in, int64_t m, int64_t n, uint8_t* dense, int64_t ld,
              void* stream) {
  if (!valid_field(field)) return fail(SG_EINVAL, "unknown field code");
  if (m < 0 || n < 0 || ld < n) return fail(SG_EINVAL, "bad shape or leading dimension");
  if (m == 0 || n == 0) return SG_OK;
  if (!dense || !planes_in) return fail(SG_EINVAL, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e;
  int* flag = flag_for(dev, &e);
  if (!flag) return cuda_fail(e, "sg_unpack flag");
  SG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st), "sg_unpack");
  SG_CUDA(launch_unpack(field, planes_in, m, n, dense, ld, flag, st), "sg_unpack launch");
  g_launches++;
  int h = 0;
  SG_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "sg_unpack");
  SG_CUDA(cudaStreamSynchronize(st), "sg_unpack");
  if (h) return fail(SG_EPATTERN, "illegal F3 pattern (sign without unit) in planes");
  return SG_OK;
}

int sg_reduce_canonical(int field, uint64_t* p, int64_t rows, int64_t n, void* stream) {
  if (!valid_field(field)) return fail(SG_EINVAL, "unknown field code");
  if (rows < 0 || n < 0) return fail(SG_EINVAL, "negative dimension");
  if (rows == 0 || n == 0 || (field != SG_F5 && field != SG_F7)) return SG_OK;
  if (!p) return fail(SG_EINVAL, "null pointer");
  SG_CUDA(launch_canonicalize(field, p, rows, w64_of(n), (cudaStream_t)stream), "sg_reduce_canonical");
  g_launches++;
  return SG_OK;
}

static int op_plane_count(int op) {
  switch (op) {
    case SG_OP_F2_ADD: return 1;
    case SG_OP_F3_ADD: case SG_OP_F3_SUB: case SG_OP_F3_NEG: case SG_OP_GF4_ADD: case SG_OP_GF4_MULX:
    case SG_OP_SCALAR_MUL_F3: case SG_OP_SCALAR_MUL_GF4: case SG_OP_Z4_ADD: case SG_OP_Z4_SUB:
    case SG_OP_Z4_NEG: case SG_OP_SCALAR_MUL_Z4: return 2;
    default: return 3;
  }
}

static bool fill_planes(Planes* out, const uint64_t* const* arr, int R) {
  out->p[0] = out->p[1] = out->p[2] = nullptr;
  if (!arr) return false;
  for (int d = 0; d < R; ++d) {
    if (!arr[d]) return false;
    out->p[d] = const_cast<uint64_t*>(arr[d]);
  }
  return true;
}

int sg_plane_op(int op, uint64_t* const* dst, const uint64_t* const* src, int64_t rows, int64_t words,
                uint64_t tail, int scalar, void* stream) {
  if (op < SG_OP_F2_ADD || op > SG_OP_SCALAR_MUL_GF8) return fail(SG_EINVAL, "unknown plane op");
  if (rows < 0 || words < 0) return fail(SG_EINVAL, "negative dimension");
  if (rows == 0 || words == 0) return SG_OK;
  const bool unary = op == SG_OP_F3_NEG || op == SG_OP_F5_NEG || op == SG_OP_F5_DOUBLE ||
                     op == SG_OP_F5_REDUCE || op == SG_OP_F7_NEG || op == SG_OP_F7_DOUBLE ||
                     op == SG_OP_F7_REDUCE || op == SG_OP_GF4_MULX ||
                     (op >= SG_OP_SCALAR_MUL_F3 && op <= SG_OP_SCALAR_MUL_GF4) || op == SG_OP_Z4_NEG ||
                     op == SG_OP_Z8_NEG || op == SG_OP_GF8_MULX || op >= SG_OP_SCALAR_MUL_Z4;
  const int R = op_plane_count(op);
  Planes d, s;
  if (!fill_planes(&d, (const uint64_t* const*)dst, R)) return fail(SG_EINVAL, "null dst plane");
  if (!unary && !fill_planes(&s, src, op == SG_OP_F5_FOLD5 ? 1 : R)) return fail(SG_EINVAL, "null src plane");
  if (unary) s.p[0] = s.p[1] = s.p[2] = nullptr;
  SG_CUDA(launch_plane_op(op, d, s, rows, words, tail, scalar, (cudaStream_t)stream), "sg_plane_op");
  g_launches++;
  return SG_OK;
}

int64_t sg_m4rm_workspace_bytes(int field, int64_t m, int64_t l, int64_t n, int k) {
  if (check_mul_args(field, (void*)1, (void*)1, (void*)1, m, l, n, k) != SG_OK) return -1;
  if (m == 0 || n == 0 || l == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  Plan p;
  if (make_plan(field, m, l, n, k, dev, &p) != SG_OK) return -1;
  return workspace_bytes_for(p, field);
}

int sg_plan(int field, int64_t m, int64_t l, int64_t n, int k, int* rows_per_cta, int* splits, int* ctas,
            int* kernel_index, int* pipelined, int* threads) {
  int rc = check_mul_args(field, (void*)1, (void*)1, (void*)1, m, l, n, k);
  if (rc != SG_OK) return rc;
  if (m == 0 || n == 0 || l == 0) return fail(SG_EINVAL, "empty product has no plan");
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  Plan p;
  rc = make_plan(field, m, l, n, k, dev, &p);
  if (rc != SG_OK) return rc;
  if (rows_per_cta) *rows_per_cta = p.ki->rt * p.ki->threads;
  if (splits) *splits = p.streamk ? -1 : p.splits;
  if (ctas) *ctas = (int)(p.grid.x * p.grid.y * p.grid.z);
  if (kernel_index) *kernel_index = p.kernel_index;
  if (pipelined) *pipelined = p.ki->sched;
  if (threads) *threads = p.ki->threads;
  return SG_OK;
}

int sg_m4rm(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l, int64_t n,
            int k, void* workspace, int64_t workspace_bytes, void* stream) {
  return m4rm_device(field, A, B, C, m, l, n, k, workspace, workspace_bytes, (cudaStream_t)stream, nullptr);
}

}  // extern "C"

namespace {
int m4rm_device(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l, int64_t n,
                int k, void* workspace, int64_t workspace_bytes, cudaStream_t stream, const StreamIn* sin) {
  int rc = check_mul_args(field, A, B, C, m, l, n, k);
  if (rc != SG_OK) return rc;
  cudaStream_t st = stream;
  const int R = planes(field);
  if (m == 0 || n == 0) return SG_OK;
  if (l == 0) {  // empty inner dimension: C = 0
    SG_CUDA(cudaMemsetAsync(C, 0, (size_t)R * m * w64_of(n) * 8, st), "sg_m4rm zero");
    return SG_OK;
  }
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev), "sg_m4rm");
  std::lock_guard<std::mutex> lk(g_mu);
  Plan p;
  rc = make_plan(field, m, l, n, k, dev, &p);
  if (rc != SG_OK) return rc;
  const int* perm = nullptr;
  if (sin) {
    // streamed B: the plan must be one the builder warps can pace (streamable) and its group
    // order must have been uploaded beforehand (prepare_streamed: no allocation may happen
    // while a streamed product waits for its chunks)
    auto it = g_perm.find(perm_key(p, dev, m, l, n));
    if (!streamable(p) || it == g_perm.end()) return fail(SG_EINVAL, "product is not prepared for streamed B");
    perm = it->second;
  }
  const int64_t need = workspace_bytes_for(p, field);
  char* ws = (char*)workspace;
  if (ws) {
    if (workspace_bytes < need) return fail(SG_EINVAL, "workspace too small (see sg_m4rm_workspace_bytes)");
  } else {
    cudaError_t e;
    ws = (char*)workspace_for(dev, st, (size_t)need, &e);
    if (!ws) return cuda_fail(e, "sg_m4rm workspace");
  }
  uint32_t* AT = (uint32_t*)ws;
  int64_t at_bytes = ((int64_t)p.at_planes * p.at_words * p.mpad * 4 + 255) / 256 * 256;
  uint32_t* partial = (p.splits > 1 || p.streamk) ? (uint32_t*)(ws + at_bytes) : nullptr;

  cudaEvent_t ev[4];
  if (g_timing)
    for (int i = 0; i < 4; ++i) cudaEventCreate(&ev[i]);
  if (g_timing) cudaEventRecord(ev[0], st);
  SG_CUDA(launch_transpose_a(field, p.K, (const uint32_t*)A, AT, m, p.mpad, p.wa32, p.at_words, st),
          "sg_m4rm index pre-pass");
  g_launches++;
  if (g_timing) cudaEventRecord(ev[1], st);
  M4rmArgs a;
  CUtensorMap tmB;
  memset(&tmB, 0, sizeof(tmB));
  a.B = (const uint32_t*)B;
  a.AT = AT;
  a.C = p.splits > 1 ? partial : (uint32_t*)C;
  a.m = m;
  a.l = l;
  a.mpad = p.mpad;
  a.wa32 = p.at_words;
  a.wc32 = p.wc32;
  a.nblocks = p.nblocks;
  a.bps = p.bps;
  a.partial = p.splits > 1;
  a.early_trigger = pdl_mode() == 2;
  {
    // B staging: one TMA tensor copy per k-block for the warp-specialized schedule (its builder
    // warps wait on an mbarrier), cp.async for the others (measured equal or better there).
    // Experiments: SG_TMA=0 stages with cp.async everywhere.
    static const int tma_env = [] {
      const char* e = getenv("SG_TMA");
      return e ? atoi(e) : -1;
    }();
    a.tma_b = tma_env != 0 && p.ki->sched == 2 && p.K == 8 && p.wc32 % 4 == 0 && ((uintptr_t)B % 16) == 0 &&
              encode_b_map(&tmB, B, field, l, p.wc32);
    // A's index words by TMA too, except under stream-K (measured: F3 32768^3 -1 %, F7 -1.4 %,
    // GF(4) 8192^3 stream-K +2.6 %; SG_TMA=2 forces it, for experiments)
    a.tma_a = a.tma_b && (tma_env == 2 || !p.streamk);
  }
  if (sin && !a.tma_b) return fail(SG_EINVAL, "streamed B needs the TMA staging path");
  a.streamk = p.streamk;
  a.units = p.units;
  a.slabs = p.slabs;
  a.P2 = p.streamk ? partial : nullptr;
  if (p.streamk) a.C = (uint32_t*)C;
  if (sin) {
    M4rmStreamArgs sa;
    static_cast<M4rmArgs&>(sa) = a;
    sa.ready = sin->ready;
    sa.epoch = sin->epoch;
    sa.first_groups = sin->first_groups;
    sa.nchunks = sin->nchunks;
    sa.perm = perm;
    sa.ngroups = p.nblocks / 4;
    sa.err = sin->err;
    SG_CUDA(launch_m4rm_streamed(*p.ki, sa, tmB, p.grid, st), "sg_m4rm streamed kernel");
  } else {
    SG_CUDA(launch_m4rm(*p.ki, a, tmB, p.grid, st), "sg_m4rm kernel");
  }
  g_launches++;
  if (g_timing) cudaEventRecord(ev[2], st);
  if (p.streamk) {
    SG_CUDA(launch_reduce_streamk(field, partial, (uint32_t*)C, m, p.wc32, p.rows, p.slabs, p.tiles, p.nblocks,
                                  p.units, (int)p.grid.x, st),
            "sg_m4rm stream-K reduce");
    g_launches++;
  } else if (p.splits > 1) {
    SG_CUDA(launch_reduce_splits(field, partial, (uint32_t*)C, m, p.mpad, p.wc32, p.splits, st),
            "sg_m4rm reduce");
    g_launches++;
  }
  if (g_timing) {
    cudaEventRecord(ev[3], st);
    cudaEventSynchronize(ev[3]);
    float t0 = 0, t1 = 0, t2 = 0;
    cudaEventElapsedTime(&t0, ev[0], ev[1]);
    cudaEventElapsedTime(&t1, ev[1], ev[2]);
    cudaEventElapsedTime(&t2, ev[2], ev[3]);
    g_last_ms[0] = t0;
    g_last_ms[1] = t1;
    g_last_ms[2] = t2;
    for (int i = 0; i < 4; ++i) cudaEventDestroy(ev[i]);
  }
  return SG_OK;
}

// Per-device state of the host-buffer pipeline (sg_m4rm_host).
struct Io {
  cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
  cudaEvent_t ev_in[8], ev_comp[16];
  Buf buf;
  std::mutex busy;  // one host-buffer product per device at a time (the staging buffers are shared)
  // streamed B: chunk flags [64] + error word, the call epoch, the error word's pinned host copy
  unsigned* ready = nullptr;
  unsigned epoch = 0;
  unsigned* err_host = nullptr;
  cudaStream_t flags = nullptr;  // writes the chunk flags behind the copies' events
  cudaEvent_t ev_chunk[64];
  std::map<int, bool> preloaded;  // fields whose auxiliary kernels are loaded
};
std::map<int, Io> io_state;

PFN_cuStreamWriteValue32_v11070 write_value_fn() {
  static PFN_cuStreamWriteValue32_v11070 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(f);
  }();
  return fn;
}

constexpr int MAX_BCHUNKS = 64;

// Streamed variant of the row-piece pipeline (B uploaded whole, A and C in Pr row pieces): the
// product of piece 0 is launched as soon as A's piece 0 is up and reads B's k-chunks as they
// land -- the upload stream publishes chunk j by writing the call's epoch to ready[j] right
// behind the chunk's copy (cuStreamWriteValue32, no SM involved) and the builder warps wait per
// k-block (M4rmArgs.ready), consuming each tile's k-blocks in arrival order (streamed_order).
// Later pieces find B complete.  Returns SG_EUNSUPPORTED when the product cannot stream.
int host_streamed(Io* d, char* dbuf, int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m,
                  int64_t l, int64_t n, int k, int device, int Pr) {
  const PFN_cuStreamWriteValue32_v11070 wv = write_value_fn();
  if (!wv) return SG_EUNSUPPORTED;
  const int R = planes(field);
  const int64_t wa = w64_of(l), wc = w64_of(n);
  auto rcut = [&](int r) { return m * r / Pr; };
  // everything that may allocate or synchronize happens before the first copy is queued
  {
    std::lock_guard<std::mutex> lk(g_mu);
    Plan p0;
    int rc = prepare_streamed(field, rcut(1), l, n, k, device, &p0);
    if (rc != SG_OK) return rc;
    int64_t ws_need = 0;
    for (int r = 0; r < Pr; ++r) {
      const int64_t rows = rcut(r + 1) - rcut(r);
      if (rows <= 0) continue;
      Plan q;
      if ((rc = make_plan(field, rows, l, n, k, device, &q)) != SG_OK) return rc;
      ws_need = std::max(ws_need, workspace_bytes_for(q, field));
    }
    cudaError_t e;
    if (!workspace_for(device, d->comp, (size_t)ws_need, &e)) return cuda_fail(e, "sg_m4rm_host workspace");
    if (!d->preloaded[field]) {
      SG_CUDA(preload_aux_kernels(field), "sg_m4rm_host preload");
      d->preloaded[field] = true;
    }
    if (!d->ready) {
      SG_CUDA(cudaStreamCreateWithFlags(&d->flags, cudaStreamNonBlocking), "sg_m4rm_host stream");
      for (int i = 0; i < MAX_BCHUNKS; ++i)
        SG_CUDA(cudaEventCreateWithFlags(&d->ev_chunk[i], cudaEventDisableTiming), "sg_m4rm_host event");
      SG_CUDA(cudaMalloc(&d->ready, (MAX_BCHUNKS + 1) * sizeof(unsigned)), "sg_m4rm_host flags");
      SG_CUDA(cudaMemset(d->ready, 0, (MAX_BCHUNKS + 1) * sizeof(unsigned)), "sg_m4rm_host flags");
      SG_CUDA(cudaMallocHost(&d->err_host, sizeof(unsigned)), "sg_m4rm_host flags");
      // first use of the stream memory operations while nothing waits on them
      if (wv((CUstream)d->flags, (CUdeviceptr)(d->ready + MAX_BCHUNKS), 0u, 0) != CUDA_SUCCESS) {
        cudaGetLastError();
        return SG_EUNSUPPORTED;
      }
      SG_CUDA(cudaStreamSynchronize(d->flags), "sg_m4rm_host flags");
    }
  }
  unsigned* err = d->ready + MAX_BCHUNKS;
  const unsigned epoch = ++d->epoch;
  // B chunks: whole 4-block groups (32 rows) in geometrically growing chunks, g0, 2 g0, 4 g0, ...
  // (chunk j = groups [g0 (2^j - 1), g0 (2^(j+1) - 1))): the first chunk is small so the product
  // starts early, later ones large so fewer copies pay the per-copy setup, and each arrives
  // before the product needs it (the product consumes B at a steady rate while the upload's
  // lead grows).  g0 = groups / 32 by default (F5 4096^3, tools/e2e_sweep.py: 4 of 128 groups
  // 0.716 ms, 2: 0.725, 8: 0.776; equal chunks of 8-16 groups: 0.72).
  const int64_t groups = (l + 31) / 32;
  const size_t b_bytes = (size_t)R * l * wc * 8;
  const char* g0_e = getenv("SG_HOST_BFIRST");  // experiments: groups in the first chunk
  int64_t g0 = g0_e ? atoll(g0_e) : (groups + 31) / 32;
  g0 = std::max<int64_t>(1, std::min<int64_t>(g0, groups));
  auto chunk_lo = [&](int j) { return std::min<int64_t>(groups, g0 * (((int64_t)1 << j) - 1)); };
  int nch = 1;
  while (chunk_lo(nch) < groups) ++nch;
  if (nch > MAX_BCHUNKS) return SG_EUNSUPPORTED;
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  char* cur = dbuf;
  uint64_t* dB = (uint64_t*)cur;
  cur += up(b_bytes);
  uint64_t* dAp[4];
  for (int r = 0; r < Pr; ++r) {
    dAp[r] = (uint64_t*)cur;
    cur += up((size_t)R * (rcut(r + 1) - rcut(r)) * wa * 8);
  }
  uint64_t* dC = (uint64_t*)cur;  // pieces back to back, each [R][rows][wc]
  // SG_HOST_TRACE=1 (experiments): event timestamps of the pipeline steps on stderr
  static const bool trace = getenv("SG_HOST_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  auto mark = [&](const std::string& what, cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    marks.push_back({what, e});
  };
  mark("start", d->in);
  auto upload_a = [&](int r) -> int {
    const int64_t q0 = rcut(r), rows = rcut(r + 1) - q0;
    if (rows > 0)
      SG_CUDA(cudaMemcpy2DAsync(dAp[r], rows * wa * 8, A + q0 * wa, m * wa * 8, rows * wa * 8, R,
                                cudaMemcpyHostToDevice, d->in),
              "sg_m4rm_host H2D A");
    SG_CUDA(cudaEventRecord(d->ev_in[r], d->in), "sg_m4rm_host event");
    mark("in: A piece " + std::to_string(r) + " up", d->in);
    return SG_OK;
  };
  auto product = [&](int r, const StreamIn* sin) -> int {
    const int64_t q0 = rcut(r), rows = rcut(r + 1) - q0;
    SG_CUDA(cudaStreamWaitEvent(d->comp, d->ev_in[r], 0), "sg_m4rm_host wait");
    if (rows <= 0) return SG_OK;
    uint64_t* piece = dC + (int64_t)R * q0 * wc;
    mark("comp: product " + std::to_string(r) + " queued (inputs up)", d->comp);
    int rc = m4rm_device(field, dAp[r], dB, piece, rows, l, n, k, nullptr, 0, d->comp, sin);
    if (rc != SG_OK) return rc;
    SG_CUDA(cudaEventRecord(d->ev_comp[r], d->comp), "sg_m4rm_host event");
    SG_CUDA(cudaStreamWaitEvent(d->out, d->ev_comp[r], 0), "sg_m4rm_host wait");
    mark("comp: product " + std::to_string(r) + " done", d->comp);
    SG_CUDA(cudaMemcpy2DAsync(C + q0 * wc, m * wc * 8, piece, rows * wc * 8, rows * wc * 8, R,
                              cudaMemcpyDeviceToHost, d->out),
            "sg_m4rm_host D2H C");
    mark("out: piece " + std::to_string(r) + " down", d->out);
    return SG_OK;
  };
  int rc;
  // Every upload is queued before the first product: with pageable host buffers a copy call may
  // block the host until the stream's earlier work is done, and piece 0's product must never be
  // waiting for chunk flags that are not queued yet.  Order: A's piece 0, B chunk by chunk (each
  // followed by its flag), A's other pieces.
  if ((rc = upload_a(0)) != SG_OK) return rc;
  for (int j = 0; j < nch; ++j) {
    const int64_t r0 = chunk_lo(j) * 32, rows = std::min<int64_t>(l, chunk_lo(j + 1) * 32) - r0;
    // Each flag goes out on its own stream behind its copy's event.  (Measured on B200: B's
    // chunks still arrive at ~30 GB/s against ~50 GB/s for one large copy -- every chunk pays
    // the copy setup; alternating two upload streams made the arrival order worse.)
    cudaStream_t cs = d->in;
    SG_CUDA(cudaMemcpy2DAsync(dB + r0 * wc, l * wc * 8, B + r0 * wc, l * wc * 8, rows * wc * 8, R,
                              cudaMemcpyHostToDevice, cs),
            "sg_m4rm_host H2D B");
    SG_CUDA(cudaEventRecord(d->ev_chunk[j], cs), "sg_m4rm_host event");
    SG_CUDA(cudaStreamWaitEvent(d->flags, d->ev_chunk[j], 0), "sg_m4rm_host wait");
    if (wv((CUstream)d->flags, (CUdeviceptr)(d->ready + j), epoch, 0) != CUDA_SUCCESS)
      return fail(SG_ECUDA, "sg_m4rm_host: cuStreamWriteValue32 failed");
    if (j == 0 || j == nch - 1 || j == nch / 2) mark("in: B chunk " + std::to_string(j) + " up", d->in);
  }
  for (int r = 1; r < Pr; ++r)
    if ((rc = upload_a(r)) != SG_OK) return rc;
  const StreamIn sin{d->ready, epoch, (int)g0, nch, err};
  for (int r = 0; r < Pr; ++r)
    if ((rc = product(r, r == 0 ? &sin : nullptr)) != SG_OK) return rc;
  SG_CUDA(cudaMemcpyAsync(d->err_host, err, sizeof(unsigned), cudaMemcpyDeviceToHost, d->comp), "sg_m4rm_host");
  SG_CUDA(cudaStreamSynchronize(d->out), "sg_m4rm_host sync");
  SG_CUDA(cudaStreamSynchronize(d->comp), "sg_m4rm_host sync");
  SG_CUDA(cudaStreamSynchronize(d->in), "sg_m4rm_host sync");
  SG_CUDA(cudaStreamSynchronize(d->flags), "sg_m4rm_host sync");
  if (trace) {
    fprintf(stderr, "host_streamed trace Pr=%d nch=%d\n", Pr, nch);
    for (auto& mk : marks) {
      float ms = 0;
      cudaEventElapsedTime(&ms, marks[0].second, mk.second);
      fprintf(stderr, "  %8.3f ms  %s\n", ms, mk.first.c_str());
    }
    for (auto& mk : marks) cudaEventDestroy(mk.second);
  }
  if (*d->err_host) {
    const unsigned c = *d->err_host - 1;
    cudaMemset(err, 0, sizeof(unsigned));
    return fail(SG_ECUDA, "sg_m4rm_host: a streamed product timed out waiting for B chunk " + std::to_string(c) +
                              " of " + std::to_string(nch));
  }
  g_streamed++;
  return SG_OK;
}

}  // namespace

extern "C" {

int sg_m4rm_host(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l, int64_t n,
                 int k, int device) {
  int rc = check_mul_args(field, A, B, C, m, l, n, k);
  if (rc != SG_OK) return rc;
  if (m == 0 || n == 0) return SG_OK;
  SG_CUDA(cudaSetDevice(device), "sg_m4rm_host set device");
  const int R = planes(field);
  const int64_t wa = w64_of(l), wc = w64_of(n);
  const size_t a_bytes = (size_t)R * m * wa * 8, b_bytes = (size_t)R * l * wc * 8, c_bytes = (size_t)R * m * wc * 8;
  // Pipeline over three streams (H2D, compute, D2H), measured on B200 (tools/e2e_chunks.py):
  //  * the inner dimension is cut into Pk word-aligned chunks: the multiply of chunk j (A's
  //    columns and B's rows of that chunk) starts as soon as that chunk is up, instead of after
  //    all of B;
  //  * the last chunk's product is cut into Pr row pieces: once piece r is done, the chunk
  //    partials of those rows are summed (canonical) and piece r goes down while r+1 computes.
  // Field sums are exact and F5 / F7 results canonical, so any chunking gives the same bits.
  const size_t io = a_bytes + b_bytes;
  // (B200, profiles/r01c_e2e_chunks.txt: F5 4096 best 1x2, GF(4) 8192 4x2, F7 16384x8192 4x4;
  // every product carries ~30 us of fixed cost, so small ones are not cut on k)
  int Pk = io >= ((size_t)24 << 20) ? 4 : 1;
  int Pr = c_bytes >= ((size_t)64 << 20) ? 4 : (c_bytes >= ((size_t)1 << 20) ? 2 : 1);
  if (const char* e = getenv("SG_HOST_KCHUNKS")) Pk = std::max(1, std::min(4, atoi(e)));  // experiments
  if (const char* e = getenv("SG_HOST_CHUNKS")) Pr = std::max(1, std::min(4, atoi(e)));
  Pk = (int)std::max<int64_t>(1, std::min<int64_t>(Pk, wa));  // chunks of whole 64-column words
  Pr = (int)std::max<int64_t>(1, std::min<int64_t>(Pr, m));
  if (l == 0) Pk = 1;
  // Alternatively (Pc > 1) a Pr x Pc grid of row pieces x column pieces, no k-chunks: product
  // (r, c) needs A's row piece r and B's column piece c, so it starts after 1/Pr + 1/Pc of the
  // inputs instead of all of B, and C leaves in Pr x Pc pieces.
  // (measured: F7 16384x8192x16384 4 x 4 grid 14.9 ms vs 15.5 with k-chunks, device 13.9 ms;
  // no gain below ~64 MB of C, where the smaller products lose more than the earlier start)
  int Pc = 1;
  if (c_bytes >= ((size_t)64 << 20)) {
    Pc = 4;
    if (!getenv("SG_HOST_CHUNKS")) Pr = (int)std::max<int64_t>(1, std::min<int64_t>(4, m));
  }
  if (const char* e = getenv("SG_HOST_CCHUNKS")) Pc = std::max(1, std::min(4, atoi(e)));  // experiments
  Pc = (int)std::max<int64_t>(1, std::min<int64_t>(Pc, wc));
  if (Pc > 1) Pk = 1;
  Io* d;
  char* dbuf = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    d = &io_state[device];  // std::map nodes are stable: d stays valid
  }
  std::lock_guard<std::mutex> busy(d->busy);  // held to the end of the call (after the final syncs)
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  // device layout: B chunks | A chunks (last one as row pieces) | chunk partials | last-chunk
  // pieces | C
  const size_t need = b_bytes + a_bytes + (size_t)(Pk - 1) * c_bytes + (Pk > 1 ? c_bytes : 0) + c_bytes + 32 * 256;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!d->in) {
      SG_CUDA(cudaStreamCreateWithFlags(&d->in, cudaStreamNonBlocking), "sg_m4rm_host stream");
      SG_CUDA(cudaStreamCreateWithFlags(&d->comp, cudaStreamNonBlocking), "sg_m4rm_host stream");
      SG_CUDA(cudaStreamCreateWithFlags(&d->out, cudaStreamNonBlocking), "sg_m4rm_host stream");
      for (int i = 0; i < 8; ++i)
        SG_CUDA(cudaEventCreateWithFlags(&d->ev_in[i], cudaEventDisableTiming), "sg_m4rm_host event");
      for (int i = 0; i < 16; ++i)
        SG_CUDA(cudaEventCreateWithFlags(&d->ev_comp[i], cudaEventDisableTiming), "sg_m4rm_host event");
    }
    if (d->buf.bytes < need) {
      if (d->buf.p) {
        cudaDeviceSynchronize();
        cudaFree(d->buf.p);
      }
      d->buf.p = nullptr;
      d->buf.bytes = 0;
      SG_CUDA(cudaMalloc(&d->buf.p, need), "sg_m4rm_host alloc");
      d->buf.bytes = need;
    }
    dbuf = (char*)d->buf.p;
  }
  const char* stream_e = getenv("SG_HOST_STREAM");  // experiments: 0 = upload B before the products
  if ((!stream_e || atoi(stream_e) != 0) && Pk == 1 && Pc == 1 && l > 0 && Pr <= 4) {
    rc = host_streamed(d, dbuf, field, A, B, C, m, l, n, k, device, Pr);
    if (rc != SG_EUNSUPPORTED) return rc;
  }
  if (Pc > 1) {
    // ---- Pr x Pc grid: uploads in order of first use, products row-major, pieces down as done
    uint64_t* dAr[4];
    uint64_t* dBc[4];
    uint64_t* dCrc[16];
    char* q = dbuf;
    auto rcut = [&](int r) { return m * r / Pr; };
    auto ccut = [&](int c) { return wc * c / Pc; };  // 64-bit words of C / B rows
    for (int c = 0; c < Pc; ++c) {
      dBc[c] = (uint64_t*)q;
      q += up((size_t)R * l * (ccut(c + 1) - ccut(c)) * 8);
    }
    for (int r = 0; r < Pr; ++r) {
      dAr[r] = (uint64_t*)q;
      q += up((size_t)R * (rcut(r + 1) - rcut(r)) * wa * 8);
      for (int c = 0; c < Pc; ++c) {
        dCrc[r * Pc + c] = (uint64_t*)q;
        q += up((size_t)R * (rcut(r + 1) - rcut(r)) * (ccut(c + 1) - ccut(c)) * 8);
      }
    }
    auto upload_b = [&](int c) -> int {
      const int64_t w0 = ccut(c), ww = ccut(c + 1) - w0;
      if (l && ww)
        SG_CUDA(cudaMemcpy2DAsync(dBc[c], ww * 8, B + w0, wc * 8, ww * 8, (size_t)R * l, cudaMemcpyHostToDevice, d->in),
                "sg_m4rm_host H2D B");
      SG_CUDA(cudaEventRecord(d->ev_in[c], d->in), "sg_m4rm_host event");
      return SG_OK;
    };
    auto upload_a = [&](int r) -> int {
      const int64_t r0 = rcut(r), rows = rcut(r + 1) - r0;
      if (wa && rows)
        SG_CUDA(cudaMemcpy2DAsync(dAr[r], rows * wa * 8, A + r0 * wa, m * wa * 8, rows * wa * 8, R,
                                  cudaMemcpyHostToDevice, d->in),
                "sg_m4rm_host H2D A");
      SG_CUDA(cudaEventRecord(d->ev_in[4 + r], d->in), "sg_m4rm_host event");
      return SG_OK;
    };
    if ((rc = upload_a(0)) != SG_OK) return rc;
    for (int c = 0; c < Pc; ++c)
      if ((rc = upload_b(c)) != SG_OK) return rc;
    for (int r = 1; r < Pr; ++r)
      if ((rc = upload_a(r)) != SG_OK) return rc;
    for (int r = 0; r < Pr; ++r) {
      const int64_t r0 = rcut(r), rows = rcut(r + 1) - r0;
      for (int c = 0; c < Pc; ++c) {
        const int64_t w0 = ccut(c), ww = ccut(c + 1) - w0;
        const int64_t ncols = std::min(n, (w0 + ww) * 64) - w0 * 64;
        SG_CUDA(cudaStreamWaitEvent(d->comp, d->ev_in[4 + r], 0), "sg_m4rm_host wait");
        SG_CUDA(cudaStreamWaitEvent(d->comp, d->ev_in[c], 0), "sg_m4rm_host wait");
        if (rows && ww) {
          rc = sg_m4rm(field, dAr[r], dBc[c], dCrc[r * Pc + c], rows, l, ncols, k, nullptr, 0, d->comp);
          if (rc != SG_OK) return rc;
        }
        SG_CUDA(cudaEventRecord(d->ev_comp[r * Pc + c], d->comp), "sg_m4rm_host event");
        SG_CUDA(cudaStreamWaitEvent(d->out, d->ev_comp[r * Pc + c], 0), "sg_m4rm_host wait");
        if (rows && ww)
          for (int p = 0; p < R; ++p)
            SG_CUDA(cudaMemcpy2DAsync(C + ((int64_t)p * m + r0) * wc + w0, wc * 8,
                                      dCrc[r * Pc + c] + (int64_t)p * rows * ww, ww * 8, ww * 8, rows,
                                      cudaMemcpyDeviceToHost, d->out),
                    "sg_m4rm_host D2H C");
      }
    }
    SG_CUDA(cudaStreamSynchronize(d->out), "sg_m4rm_host sync");
    SG_CUDA(cudaStreamSynchronize(d->comp), "sg_m4rm_host sync");
    SG_CUDA(cudaStreamSynchronize(d->in), "sg_m4rm_host sync");
    return SG_OK;
  }

  // SG_HOST_TRACE=1 (experiments): event timestamps of every pipeline step on stderr
  static const bool trace = getenv("SG_HOST_TRACE") != nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> marks;
  cudaEvent_t t0 = nullptr;
  if (trace) {
    cudaEventCreate(&t0);
    cudaEventRecord(t0, d->in);
  }
  auto mark = [&](const char* what, cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    marks.push_back({what, e});
  };
  char* cur = dbuf;
  auto take = [&](size_t bytes) {
    char* p = cur;
    cur += up(bytes);
    return (uint64_t*)p;
  };
  auto wcut = [&](int j) { return wa * j / Pk; };  // chunk j = words [wcut(j), wcut(j+1)) of A's rows
  auto rcut = [&](int r) { return m * r / Pr; };
  // ---- uploads: B rows and A columns of chunk j (j < Pk-1), then the last chunk by row pieces
  uint64_t* dB[4];
  uint64_t* dA[4];
  uint64_t* dAp[4];
  for (int j = 0; j < Pk; ++j) {
    const int64_t w0 = wcut(j), w1 = wcut(j + 1);
    const int64_t r0 = std::min(l, w0 * 64), r1 = j == Pk - 1 ? l : std::min(l, w1 * 64);  // B rows
    dB[j] = take((size_t)R * (r1 - r0) * wc * 8);
    if (r1 > r0)
      SG_CUDA(cudaMemcpy2DAsync(dB[j], (r1 - r0) * wc * 8, B + r0 * wc, l * wc * 8, (r1 - r0) * wc * 8, R,
                                cudaMemcpyHostToDevice, d->in),
              "sg_m4rm_host H2D B");
    if (j < Pk - 1) {
      dA[j] = take((size_t)R * m * (w1 - w0) * 8);
      // all R*m rows share the pitch wa: one 2D copy of the column range
      SG_CUDA(cudaMemcpy2DAsync(dA[j], (w1 - w0) * 8, A + w0, wa * 8, (w1 - w0) * 8, (size_t)R * m,
                                cudaMemcpyHostToDevice, d->in),
              "sg_m4rm_host H2D A");
      mark("in: chunk up", d->in);
      SG_CUDA(cudaEventRecord(d->ev_in[j], d->in), "sg_m4rm_host event");
    } else {
      for (int r = 0; r < Pr; ++r) {
        const int64_t q0 = rcut(r), q1 = rcut(r + 1);
        dAp[r] = take((size_t)R * (q1 - q0) * (w1 - w0) * 8);
        if (q1 > q0 && w1 > w0)
          for (int p = 0; p < R; ++p)
            SG_CUDA(cudaMemcpy2DAsync(dAp[r] + (int64_t)p * (q1 - q0) * (w1 - w0), (w1 - w0) * 8,
                                      A + ((int64_t)p * m + q0) * wa + w0, wa * 8, (w1 - w0) * 8, q1 - q0,
                                      cudaMemcpyHostToDevice, d->in),
                    "sg_m4rm_host H2D A");
        mark("in: last-chunk piece up", d->in);
        SG_CUDA(cudaEventRecord(d->ev_in[Pk - 1 + r], d->in), "sg_m4rm_host event");
      }
    }
  }
  // ---- products: chunk partials S_j over all rows, then the last chunk piece by piece
  uint64_t* S[4];
  for (int j = 0; j + 1 < Pk; ++j) S[j] = take(c_bytes);
  uint64_t* L = Pk > 1 ? take(c_bytes) : nullptr;  // last-chunk pieces, each [R][rows][wc]
  uint64_t* dC = take(c_bytes);                     // final C, [R][m][wc]
  for (int j = 0; j + 1 < Pk; ++j) {
    const int64_t w0 = wcut(j), w1 = wcut(j + 1);
    SG_CUDA(cudaStreamWaitEvent(d->comp, d->ev_in[j], 0), "sg_m4rm_host wait");
    rc = sg_m4rm(field, dA[j], dB[j], S[j], m, std::min(l, w1 * 64) - w0 * 64, n, k, nullptr, 0, d->comp);
    if (rc != SG_OK) return rc;
    mark("comp: chunk product", d->comp);
  }
  const int64_t lw0 = wcut(Pk - 1) * 64, l_last = l - std::min(l, lw0);
  uint64_t* Lcur = L;
  for (int r = 0; r < Pr; ++r) {
    const int64_t q0 = rcut(r), q1 = rcut(r + 1), rows = q1 - q0;
    SG_CUDA(cudaStreamWaitEvent(d->comp, d->ev_in[Pk - 1 + r], 0), "sg_m4rm_host wait");
    if (rows > 0) {
      if (Pk == 1) {
        // no chunk partials: the piece lands in C directly (rows q0.. of every plane)
        uint64_t* piece = dC + (int64_t)R * q0 * wc;  // pieces packed back to back, each [R][rows][wc]
        rc = sg_m4rm(field, dAp[r], dB[0], piece, rows, l, n, k, nullptr, 0, d->comp);
        if (rc != SG_OK) return rc;
        mark("comp: piece product", d->comp);
        SG_CUDA(cudaEventRecord(d->ev_comp[r], d->comp), "sg_m4rm_host event");
        SG_CUDA(cudaStreamWaitEvent(d->out, d->ev_comp[r], 0), "sg_m4rm_host wait");
        SG_CUDA(cudaMemcpy2DAsync(C + q0 * wc, m * wc * 8, piece, rows * wc * 8, rows * wc * 8, R,
                                  cudaMemcpyDeviceToHost, d->out),
                "sg_m4rm_host D2H C");
        mark("out: piece down", d->out);
        continue;
      }
      rc = sg_m4rm(field, dAp[r], dB[Pk - 1], Lcur, rows, l_last, n, k, nullptr, 0, d->comp);
      if (rc != SG_OK) return rc;
      SliceSet ss;
      ss.n = Pk;
      for (int j = 0; j + 1 < Pk; ++j) {
        ss.base[j] = (const uint32_t*)(S[j] + q0 * wc);
        ss.pstride[j] = 2 * m * wc;
      }
      ss.base[Pk - 1] = (const uint32_t*)Lcur;
      ss.pstride[Pk - 1] = 2 * rows * wc;
      SG_CUDA(launch_sum_slices(field, ss, (uint32_t*)(dC + q0 * wc), 2 * m * wc, rows, (int)(2 * wc), d->comp),
              "sg_m4rm_host chunk sum");
      g_launches++;
      mark("comp: piece product + sum", d->comp);
      SG_CUDA(cudaEventRecord(d->ev_comp[r], d->comp), "sg_m4rm_host event");
      SG_CUDA(cudaStreamWaitEvent(d->out, d->ev_comp[r], 0), "sg_m4rm_host wait");
      SG_CUDA(cudaMemcpy2DAsync(C + q0 * wc, m * wc * 8, dC + q0 * wc, m * wc * 8, rows * wc * 8, R,
                                cudaMemcpyDeviceToHost, d->out),
              "sg_m4rm_host D2H C");
      mark("out: piece down", d->out);
      Lcur += (int64_t)R * rows * wc;
    }
  }
  SG_CUDA(cudaStreamSynchronize(d->out), "sg_m4rm_host sync");
  SG_CUDA(cudaStreamSynchronize(d->comp), "sg_m4rm_host sync");
  SG_CUDA(cudaStreamSynchronize(d->in), "sg_m4rm_host sync");
  if (trace) {
    fprintf(stderr, "sg_m4rm_host trace Pk=%d Pr=%d\n", Pk, Pr);
    for (auto& mk : marks) {
      float ms = 0;
      cudaEventElapsedTime(&ms, t0, mk.second);
      fprintf(stderr, "  %8.3f ms  %s\n", ms, mk.first);
      cudaEventDestroy(mk.second);
    }
    cudaEventDestroy(t0);
  }
  return SG_OK;
}

int sg_m4rm_multi(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l, int64_t n,
                  int k, int ngpus, const int* devices) {
  int rc = check_mul_args(field, A, B, C, m, l, n, k);
  if (rc != SG_OK) return rc;
  if (ngpus < 1 || ngpus > 64 || !devices) return fail(SG_EINVAL, "need 1..64 devices");
  int ndev = 0;
  SG_CUDA(cudaGetDeviceCount(&ndev), "sg_m4rm_multi device count");
  for (int g = 0; g < ngpus; ++g)
    if (devices[g] < 0 || devices[g] >= ndev) return fail(SG_EINVAL, "device index out of range");
  if (m == 0 || n == 0) return SG_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  const int R = planes(field);
  const int64_t wa = w64_of(l), wc = w64_of(n);
  const size_t b_bytes = (size_t)R * l * wc * 8;
  struct Dev {
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    Buf buf;
  };
  static std::map<int, Dev> state;
  static std::mutex multi_mu;
  std::lock_guard<std::mutex> busy(multi_mu);  // one multi-device product at a time
  // per distinct device: B, then the A and C slabs of every shard it runs
  std::map<int, size_t> need;
  std::vector<int64_t> r0(ngpus), r1(ngpus);
  for (int g = 0; g < ngpus; ++g) {
    r0[g] = m * g / ngpus;
    r1[g] = m * (g + 1) / ngpus;
    need[devices[g]] += ((size_t)R * (r1[g] - r0[g]) * (wa + wc) * 8 + 2 * 256);
  }
  for (auto& kv : need) {
    kv.second += b_bytes + 256;
    Dev& d = state[kv.first];
    SG_CUDA(cudaSetDevice(kv.first), "sg_m4rm_multi set device");
    if (!d.st) {
      SG_CUDA(cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking), "sg_m4rm_multi stream");
      SG_CUDA(cudaEventCreateWithFlags(&d.ev, cudaEventDisableTiming), "sg_m4rm_multi event");
    }
    if (d.buf.bytes < kv.second) {
      if (d.buf.p) {
        cudaDeviceSynchronize();
        cudaFree(d.buf.p);
      }
      d.buf.p = nullptr;
      d.buf.bytes = 0;
      SG_CUDA(cudaMalloc(&d.buf.p, kv.second), "sg_m4rm_multi alloc");
      d.buf.bytes = kv.second;
    }
  }
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  // B: host -> devices[0], then peer copies to every other device (one hop each over NVSwitch)
  const int d0 = devices[0];
  uint64_t* B0 = (uint64_t*)state[d0].buf.p;
  SG_CUDA(cudaSetDevice(d0), "sg_m4rm_multi set device");
  if (b_bytes) SG_CUDA(cudaMemcpyAsync(B0, B, b_bytes, cudaMemcpyHostToDevice, state[d0].st), "sg_m4rm_multi H2D B");
  SG_CUDA(cudaEventRecord(state[d0].ev, state[d0].st), "sg_m4rm_multi event");
  for (auto& kv : need) {
    if (kv.first == d0 || !b_bytes) continue;
    Dev& d = state[kv.first];
    SG_CUDA(cudaSetDevice(kv.first), "sg_m4rm_multi set device");
    int can = 0;
    cudaDeviceCanAccessPeer(&can, kv.first, d0);
    if (can) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(d0, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "sg_m4rm_multi peer access");
      cudaGetLastError();
    }
    SG_CUDA(cudaStreamWaitEvent(d.st, state[d0].ev, 0), "sg_m4rm_multi wait");
    SG_CUDA(cudaMemcpyPeerAsync(d.buf.p, kv.first, B0, d0, b_bytes, d.st), "sg_m4rm_multi peer copy B");
  }
  // shards: A rows up, multiply, C rows down (each device's stream; shards on one device in order)
  std::map<int, size_t> offset;
  for (auto& kv : need) offset[kv.first] = up(b_bytes);
  for (int g = 0; g < ngpus; ++g) {
    const int dv = devices[g];
    Dev& d = state[dv];
    const int64_t rows = r1[g] - r0[g];
    if (rows == 0) continue;
    SG_CUDA(cudaSetDevice(dv), "sg_m4rm_multi set device");
    char* base = (char*)d.buf.p;
    uint64_t* dB = (uint64_t*)base;
    uint64_t* dA = (uint64_t*)(base + offset[dv]);
    offset[dv] += up((size_t)R * rows * wa * 8);
    uint64_t* dC = (uint64_t*)(base + offset[dv]);
    offset[dv] += up((size_t)R * rows * wc * 8);
    if (wa)
      SG_CUDA(cudaMemcpy2DAsync(dA, rows * wa * 8, A + r0[g] * wa, m * wa * 8, rows * wa * 8, R,
                                cudaMemcpyHostToDevice, d.st),
              "sg_m4rm_multi H2D A");
    rc = sg_m4rm(field, dA, dB, dC, rows, l, n, k, nullptr, 0, d.st);
    if (rc != SG_OK) {
      cudaSetDevice(cur);
      return rc;
    }
    SG_CUDA(cudaMemcpy2DAsync(C + r0[g] * wc, m * wc * 8, dC, rows * wc * 8, rows * wc * 8, R,
                              cudaMemcpyDeviceToHost, d.st),
            "sg_m4rm_multi D2H C");
  }
  for (auto& kv : need) {
    SG_CUDA(cudaSetDevice(kv.first), "sg_m4rm_multi set device");
    SG_CUDA(cudaStreamSynchronize(state[kv.first].st), "sg_m4rm_multi sync");
  }
  cudaSetDevice(cur);
  return SG_OK;
}

int sg_build_table(int field, const uint64_t* const* B, int64_t b_rows, int64_t row_base, int kp, int64_t words,
                   uint64_t* const* T, void* stream) {
  if (!valid_field(field)) return fail(SG_EINVAL, "unknown field code");
  if (kp < 0 || kp > 16 || row_base < 0 || words < 0 || b_rows < 0) return fail(SG_EINVAL, "bad table shape");
  Planes b, t;
  if (!fill_planes(&b, B, planes(field)) || !fill_planes(&t, (const uint64_t* const*)T, planes(field)))
    return fail(SG_EINVAL, "null plane pointer");
  SG_CUDA(launch_build_table(field, b, b_rows, row_base, kp, words, t, (cudaStream_t)stream), "sg_build_table");
  g_launches++;
  return SG_OK;
}

int sg_m4rm_block(int field, uint64_t* const* C, int64_t c_words, const uint64_t* const* A, int64_t a_words,
                  int64_t col0, int kp, const uint64_t* const* T, int64_t row0, int64_t row1, void* stream) {
  if (!valid_field(field)) return fail(SG_EINVAL, "unknown field code");
  if (kp < 0 || kp > 16 || col0 < 0 || row0 < 0 || row1 < row0) return fail(SG_EINVAL, "bad block arguments");
  if (col0 + kp > a_words * 64) return fail(SG_EINVAL, "block exceeds A's columns");
  if (row1 == row0 || c_words == 0 || kp == 0) return SG_OK;
  Planes c, a, t;
  const int R = planes(field);
  if (!fill_planes(&c, (const uint64_t* const*)C, R) || !fill_planes(&a, A, R) || !fill_planes(&t, T, R))
    return fail(SG_EINVAL, "null plane pointer");
  SG_CUDA(launch_block_driver(field, c, c_words, a, a_words, col0, kp, t, row0, row1, (cudaStream_t)stream),
          "sg_m4rm_block");
  g_launches++;
  return SG_OK;
}

int sg_classical(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l, int64_t n,
                 void* stream) {
  int rc = check_mul_args(field, A, B, C, m, l, n, 1);
  if (rc != SG_OK) return rc;
  if (m == 0 || n == 0) return SG_OK;
  const int R = planes(field);
  const int64_t wa = w64_of(l), wb = w64_of(n);
  if (l == 0) {
    SG_CUDA(cudaMemsetAsync(C, 0, (size_t)R * m * wb * 8, (cudaStream_t)stream), "sg_classical zero");
    return SG_OK;
  }
  Planes a, b, c;
  for (int d = 0; d < 3; ++d) {
    a.p[d] = d < R ? const_cast<uint64_t*>(A) + d * m * wa : nullptr;
    b.p[d] = d < R ? const_cast<uint64_t*>(B) + d * l * wb : nullptr;
    c.p[d] = d < R ? C + d * m * wb : nullptr;
  }
  SG_CUDA(launch_classical(field, a, wa, b, wb, c, m, l, (cudaStream_t)stream), "sg_classical");
  g_launches++;
  return SG_OK;
}

int sg_probe_peaks(int device, double* lop3, double* lds, double* mhz) {
  if (!lop3 || !lds || !mhz) return fail(SG_EINVAL, "null pointer");
  if (probe_peaks(device, lop3, lds, mhz) != 0) return fail(SG_ECUDA, "peak probe failed");
  g_launches += 6;
  return SG_OK;
}

}  // extern "C"

// sg_api.cu -- the C ABI (include/slicegemm_b200.h): library state and errors, argument checks,
// workspace management, one product on device buffers (m4rm_device), timing and launch
// accounting, and the block-granularity plugin mirror.  The planner is sg_plan.cu, the
// host-buffer pipelines sg_host.cu.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <cudaTypedefs.h>

#include "sg_api_internal.h"
#include "sg_field.cuh"

namespace sg {
namespace api {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_buffer_generation{0};
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



// ---------------------------------------------------------------- per-device state
std::map<int, DevState> g_dev;

DevState& dev_state(int device) {
  DevState& d = g_dev[device];
  if (!d.attrs_set) {
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device);
    for (int i = 0; i < m4rm_kernel_count(); ++i) {
      KernelInfo* k = m4rm_kernel_at(i);
      const void* fn = k->fn ? (const void*)k->fn : (const void*)k->fn_fused;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem_bytes);
      if (k->fn_stream &&
          cudaFuncSetAttribute(k->fn_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem_stream) != cudaSuccess)
        k->fn_stream = nullptr;  // does not fit this device: no streamed variant
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess) k->regs = fa.numRegs;
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, k->launch_threads, k->smem_bytes);
      k->occupancy = occ;
    }
    cudaGetLastError();
    d.attrs_set = true;
  }
  return d;
}

// Workspace cache keyed by (device, stream): stream-ordered reuse is safe, cross-stream is not.
std::map<std::pair<int, cudaStream_t>, Buf> g_ws;
// Input-check status of sg_pack / sg_unpack, per (device, stream): a word of mapped page-locked
// host memory that the kernels OR their error bits into (1: entry out of range, 2: illegal F3
// pattern) -- only when they find bad input, so the check costs nothing on good input and
// nothing waits for it.  sg_stream_check synchronizes the stream and reads and clears it.
std::mutex g_flag_mu;  // never held across a synchronization
std::map<std::pair<int, cudaStream_t>, StatusFlag> g_flags;

StatusFlag* flag_for(int device, cudaStream_t st, cudaError_t* err) {
  std::lock_guard<std::mutex> lk(g_flag_mu);
  StatusFlag& f = g_flags[{device, st}];
  *err = cudaSuccess;
  if (!f.host) {
    *err = cudaHostAlloc((void**)&f.host, sizeof(int), cudaHostAllocMapped);
    if (*err != cudaSuccess) {
      f.host = nullptr;
      return nullptr;
    }
    *f.host = 0;
    *err = cudaHostGetDevicePointer((void**)&f.dev, f.host, 0);
    if (*err != cudaSuccess) {
      cudaFreeHost(f.host);
      f.host = nullptr;
      return nullptr;
    }
  }
  return &f;
}

// Split-K arrival / departure counters of the fused small-product kernel, per (device, stream):
// zeroed once, and every fused launch leaves them zero (M4rmFusedArgs).
std::map<std::pair<int, cudaStream_t>, Buf> g_cnt;
unsigned* fused_counters(int device, cudaStream_t st, int ntiles, cudaError_t* err) {
  Buf& b = g_cnt[{device, st}];
  *err = cudaSuccess;
  const size_t bytes = (size_t)2 * std::max(ntiles, 4096) * sizeof(unsigned);
  if (b.bytes < bytes) {
    if (b.p) {
      cudaStreamSynchronize(st);
      cudaFree(b.p);
    }
    b.p = nullptr;
    b.bytes = 0;
    g_buffer_generation++;
    if ((*err = cudaMalloc(&b.p, bytes)) != cudaSuccess) return nullptr;
    if ((*err = cudaMemsetAsync(b.p, 0, bytes, st)) != cudaSuccess) return nullptr;
    b.bytes = bytes;
  }
  return (unsigned*)b.p;
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
    g_buffer_generation++;
    *err = cudaMalloc(&b.p, bytes);
    if (*err != cudaSuccess) return nullptr;
    b.bytes = bytes;
  }
  return b.p;
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
    perm = streamed_order_on_device(p, dev, m, l, n);
    if (!streamable(p) || !perm) return fail(SG_EINVAL, "product is not prepared for streamed B");
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
  if (p.ki->fn_fused) {
    // one cooperative launch: A's words staged directly, split-K summed in the kernel
    if (sin) return fail(SG_EINVAL, "product is not prepared for streamed B");
    M4rmFusedArgs fa;
    memset(&fa, 0, sizeof(fa));
    fa.B = (const uint32_t*)B;
    fa.AT = nullptr;
    fa.A = (const uint32_t*)A;
    fa.C = (uint32_t*)C;  // splits == 1: C directly; else compact slots in P2, summed into Cout
    fa.P2 = p.splits > 1 ? partial : nullptr;
    fa.Cout = (uint32_t*)C;
    fa.m = m;
    fa.l = l;
    fa.mpad = p.mpad;
    fa.wa32 = p.wa32;
    fa.wc32 = p.wc32;
    fa.nblocks = p.nblocks;
    fa.bps = p.bps;
    fa.partial = p.splits > 1;
    fa.ntiles = (int)(p.grid.x * p.grid.y);
    cudaError_t e;
    fa.cnt = fa.partial ? fused_counters(dev, st, fa.ntiles, &e) : nullptr;
    if (fa.partial && !fa.cnt) return cuda_fail(e, "sg_m4rm fused counters");
    CUtensorMap tmB;
    memset(&tmB, 0, sizeof(tmB));
    cudaEvent_t ev[2];
    if (g_timing) {
      for (int i = 0; i < 2; ++i) cudaEventCreate(&ev[i]);
      cudaEventRecord(ev[0], st);
    }
    SG_CUDA(launch_m4rm_fused(*p.ki, fa, tmB, p.grid, st), "sg_m4rm fused kernel");
    g_launches++;
    if (g_timing) {
      cudaEventRecord(ev[1], st);
      cudaEventSynchronize(ev[1]);
      float t1 = 0;
      cudaEventElapsedTime(&t1, ev[0], ev[1]);
      g_last_ms[0] = 0;
      g_last_ms[1] = t1;
      g_last_ms[2] = 0;
      for (int i = 0; i < 2; ++i) cudaEventDestroy(ev[i]);
    }
    return SG_OK;
  }

  cudaEvent_t ev[4];
  if (g_timing)
    for (int i = 0; i < 4; ++i) cudaEventCreate(&ev[i]);
  if (g_timing) cudaEventRecord(ev[0], st);
  SG_CUDA(launch_transpose_a(field, p.K, (const uint32_t*)A, AT, m, p.mpad, p.wa32, p.at_words, p.ki->pair_nt, st),
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
    a.tma_b = tma_env != 0 && ws_tma(p.ki->sched) && p.K == 8 && p.wc32 % 4 == 0 && ((uintptr_t)B % 16) == 0 &&
              encode_b_map(&tmB, B, field, l, p.wc32);
    // A's index words by TMA too, except under stream-K for F3 / F5 / F7 (measured: F3 32768^3
    // -1 %, F7 -1.4 %); GF(4)'s Karatsuba kernel, whose builder warps are its critical path
    // (three replicated table planes), gains 3.9 % (1.349 -> 1.297 ms).  SG_TMA=2 forces it.
    // (schedule 6 stages the index words just in time where it has two slots: TMA keeps the
    // builders from waiting on their own cp.async group)
    a.tma_a = a.tma_b && (tma_env == 2 || !p.streamk || field == SG_GF4 || p.ki->sched == 6);
  }
  if (sin && !a.tma_b) return fail(SG_EINVAL, "streamed B needs the TMA staging path");
  a.streamk = p.streamk;
  a.units = p.units;
  a.dp_tiles = p.dp_tiles;
  a.slabs = p.slabs;
  a.P2 = p.streamk ? partial : nullptr;
  if (p.streamk) a.C = (uint32_t*)C;
  if (sin) {
    M4rmStreamArgs sa;
    static_cast<M4rmArgs&>(sa) = a;
    sa.ready = sin->ready;
    sa.epoch = sin->epoch;
    sa.first_groups = sin->first_groups;
    sa.cap_log = sin->cap_log;
    sa.nchunks = sin->nchunks;
    sa.poll_ns = sin->poll_ns;
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
    SG_CUDA(launch_reduce_streamk(field, partial, (uint32_t*)C, m, p.wc32, p.rows, p.slabs, p.tiles - p.dp_tiles,
                                  p.dp_tiles, p.nblocks, p.units, (int)p.grid.x, st),
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

}  // namespace api
}  // namespace sg

using namespace sg;
using namespace sg::api;

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
  if (schedule) *schedule = ki->sched + (ki->fn_fused ? SCHED_FUSED : 0);
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

#ifdef SG_EXPERIMENTS
// performance experiments only (tools/ablate.py, `make EXTRA=-DSG_EXPERIMENTS`): select kernel
// variants with parts of the work removed; every product is WRONG while a nonzero mask is set.
// Not declared in include/slicegemm_b200.h and not compiled into the production library.
extern "C" int sg_debug_ablation(int mask) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_ablation = mask;
  return SG_OK;
}
#endif

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
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev), "sg_pack");
  cudaError_t e;
  StatusFlag* flag = flag_for(dev, st, &e);
  if (!flag) return cuda_fail(e, "sg_pack status flag");
  SG_CUDA(launch_pack(field, dense, m, n, ld, planes_out, flag->dev, st), "sg_pack launch");
  g_launches++;
  return SG_OK;  // an out-of-range entry is reported by sg_stream_check
}

int sg_unpack(int field, const uint64_t* planes_in, int64_t m, int64_t n, uint8_t* dense, int64_t ld,
              void* stream) {
  if (!valid_field(field)) return fail(SG_EINVAL, "unknown field code");
  if (m < 0 || n < 0 || ld < n) return fail(SG_EINVAL, "bad shape or leading dimension");
  if (m == 0 || n == 0) return SG_OK;
  if (!dense || !planes_in) return fail(SG_EINVAL, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev), "sg_unpack");
  cudaError_t e;
  StatusFlag* flag = flag_for(dev, st, &e);
  if (!flag) return cuda_fail(e, "sg_unpack status flag");
  SG_CUDA(launch_unpack(field, planes_in, m, n, dense, ld, flag->dev, st), "sg_unpack launch");
  g_launches++;
  return SG_OK;  // an illegal F3 pattern is reported by sg_stream_check
}

int sg_stream_check(void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev), "sg_stream_check");
  SG_CUDA(cudaStreamSynchronize(st), "sg_stream_check");
  int bits = 0;
  {
    std::lock_guard<std::mutex> lk(g_flag_mu);
    auto it = g_flags.find({dev, st});
    if (it != g_flags.end() && it->second.host) {
      bits = *(volatile int*)it->second.host;
      *(volatile int*)it->second.host = 0;
    }
  }
  if (bits & 1) return fail(SG_ERANGE, "sg_pack: entries out of range for the field");
  if (bits & 2) return fail(SG_EPATTERN, "sg_unpack: illegal F3 pattern (sign without unit) in planes");
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
  if (pipelined) *pipelined = p.ki->sched + (p.ki->fn_fused ? SCHED_FUSED : 0);
  if (threads) *threads = p.ki->threads;
  return SG_OK;
}

int sg_m4rm(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l, int64_t n,
            int k, void* workspace, int64_t workspace_bytes, void* stream) {
  return m4rm_device(field, A, B, C, m, l, n, k, workspace, workspace_bytes, (cudaStream_t)stream, nullptr);
}

}  // extern "C"

extern "C" {

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

int sg_classical_block(int field, uint64_t* const* C, int64_t c_words, const uint64_t* const* A, int64_t a_words,
                       const uint64_t* const* B, int64_t m, int64_t l, void* stream) {
  if (!valid_field(field)) return fail(SG_EINVAL, "unknown field code");
  if (m < 0 || l < 0 || c_words < 0 || a_words < 0) return fail(SG_EINVAL, "negative dimension");
  if (l > a_words * 64) return fail(SG_EINVAL, "A has fewer columns than B has rows");
  if (m == 0 || l == 0 || c_words == 0) return SG_OK;
  Planes c, a, b;
  const int R = planes(field);
  if (!fill_planes(&c, (const uint64_t* const*)C, R) || !fill_planes(&a, A, R) || !fill_planes(&b, B, R))
    return fail(SG_EINVAL, "null plane pointer");
  SG_CUDA(launch_classical_block(field, c, c_words, a, a_words, b, m, l, (cudaStream_t)stream), "sg_classical_block");
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

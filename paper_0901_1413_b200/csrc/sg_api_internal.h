// sg_api_internal.h -- host-side internals shared by sg_api.cu (C ABI, workspaces, device
// products), sg_plan.cu (launch planner, streamed-B group order) and sg_host.cu (host-buffer
// pipelines, single-process multi-GPU).
#pragma once
#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/slicegemm_b200.h"
#include "sg_internal.h"

namespace sg {
namespace api {

// ---- library state (sg_api.cu)
extern thread_local std::string g_err;
extern std::atomic<int64_t> g_launches;
// bumped whenever a library-owned device buffer (workspace, fused counters) is reallocated:
// captured graphs that baked the old pointer in must be dropped (sg_host.cu)
extern std::atomic<int64_t> g_buffer_generation;
extern std::atomic<int64_t> g_streamed;  // host-buffer products that streamed B (sg_host_streamed_count)
extern int g_override_rt, g_override_splits, g_override_pipe, g_override_threads, g_ablation;
extern int g_sm_reserve;  // SMs the planner leaves free (for a collective running concurrently)
extern bool g_timing;
extern double g_last_ms[3];
extern std::mutex g_mu;

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
#define SG_CUDA(call, where)                            \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

inline bool valid_field(int f) { return f >= SG_F2 && f <= SG_Z8; }
inline int planes(int f) { return f == SG_F2 ? 1 : (f == SG_F5 || f == SG_F7 || f == SG_GF8 || f == SG_Z8) ? 3 : 2; }
inline int64_t w64_of(int64_t n) { return (n + 63) / 64; }

// ---- per-device state and workspaces (sg_api.cu)
struct DevState {
  bool attrs_set = false;
  int sms = 148;
};

DevState& dev_state(int device);

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct StatusFlag {
  int* host = nullptr;  // mapped page-locked word (sg_stream_check reads it)
  int* dev = nullptr;   // its device alias (the kernels write it)
};
StatusFlag* flag_for(int device, cudaStream_t st, cudaError_t* err);
void* workspace_for(int device, cudaStream_t st, size_t bytes, cudaError_t* err);
int check_mul_args(int field, const void* A, const void* B, const void* C, int64_t m, int64_t l, int64_t n, int k);

// ---- planner (sg_plan.cu)
struct Plan {
  KernelInfo* ki = nullptr;
  int kernel_index = -1;
  int K = 8, splits = 1, bps = 0, nblocks = 0;
  int64_t mpad = 0;
  int wa32 = 0, wc32 = 0;
  int at_words = 0, at_planes = 0;  // staged index array: k=8 packed words (1 plane), else A^T planes
  bool streamk = false;              // one wave of CTAs over tiles x k-blocks (see m4rm_kernel)
  int64_t units = 0, tiles = 0;
  int64_t dp_tiles = 0;              // stream-K hybrid: leading tiles processed whole (units cover the rest)
  int slabs = 0, rows = 0;
  dim3 grid;
  double est_clk = 0;
};

// Measured per-CTA cost of the k = 8 variants on B200 (tools/tune.py over BASELINE.json's configs
// and the per-rank shapes of the sharded runs, fitted by tools/fit_calib.py to the model below;
// profiles/r01d_tune_all.jsonl): {field, rows per thread, lookup threads, schedule, clocks per
// k-block, clocks per CTA}.
int make_plan(int field, int64_t m, int64_t l, int64_t n, int k, int device, Plan* out);
bool encode_b_map(CUtensorMap* map, const void* B, int field, int64_t l, int wc32);
int64_t workspace_bytes_for(const Plan& p, int field);

// ---- streamed B (sg_plan.cu: group order; sg_host.cu: the pipeline)
// A product whose B arrives chunk by chunk while it runs (see M4rmArgs.ready).
struct StreamIn {
  const unsigned* ready;
  unsigned epoch;
  int first_groups;  // B's chunk j = 4-block groups [chunk_lo(j), chunk_lo(j + 1)) (sg_internal.h)
  int cap_log;       // chunks double from first_groups up to first_groups 2^cap_log, then stay
  int nchunks;
  unsigned poll_ns;
  unsigned* err;
};

bool streamable(const Plan& p);
int prepare_streamed(int field, int64_t m, int64_t l, int64_t n, int k, int dev, Plan* out);
// the device copy of a prepared product's group order, or nullptr (callers hold g_mu)
const int* streamed_order_on_device(const Plan& p, int dev, int64_t m, int64_t l, int64_t n);

// ---- one product on device buffers (sg_api.cu); sin = streamed B or nullptr
int m4rm_device(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l, int64_t n,
                int k, void* workspace, int64_t workspace_bytes, cudaStream_t stream, const StreamIn* sin);

}  // namespace api
}  // namespace sg

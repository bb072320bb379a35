// sg_host.cu -- host-buffer entry points: sg_m4rm_host (copies overlapped with the products on
// upload / compute / download / flag streams; the streamed-B pipeline for the shapes that allow
// it) and sg_m4rm_multi (rows of A and C split over devices, B replicated by peer copies).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <cudaTypedefs.h>

#include "sg_api_internal.h"

namespace sg {
namespace api {
namespace {

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
  int stream_ops = 0;  // cuStreamWriteValue32 on this device: 0 untested, 1 works, -1 unsupported
  // small calls (sg_m4rm_host's one-stream path) repeated on the same buffers replay a CUDA
  // graph of (H2D A, H2D B, product, D2H C): one launch instead of four plus the planner.
  // Keyed on everything the captured work depends on; dropped when the staging buffer moves.
  typedef std::tuple<int, const void*, const void*, void*, int64_t, int64_t, int64_t, int, std::vector<int>> GraphKey;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, int> graph_seen;  // calls so far (the first runs uncaptured: it allocates)
  int64_t graph_generation = -1;       // g_buffer_generation the graphs were captured under
};

// After a failed call, wait for every copy already queued on the device's pipeline streams: the
// caller may free or reuse its host buffers as soon as the call returns.
void drain(Io* d) {
  for (cudaStream_t s : {d->in, d->flags, d->comp, d->out})
    if (s) cudaStreamSynchronize(s);
  cudaGetLastError();
}
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
// land -- an event behind chunk j's copy releases, on the flags stream, a cuStreamWriteValue32 of
// the call's epoch into ready[j] (no SM involved), and the builder warps wait per k-block
// (M4rmStreamArgs.ready), consuming each tile's k-blocks in arrival order (streamed_order).
// Later pieces find B complete.  Returns SG_EUNSUPPORTED when the product cannot stream.
int host_streamed(Io* d, char* dbuf, int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m,
                  int64_t l, int64_t n, int k, int device, int Pr) {
  const PFN_cuStreamWriteValue32_v11070 wv = write_value_fn();
  if (!wv || d->stream_ops < 0) return SG_EUNSUPPORTED;
  const auto t_entry = std::chrono::steady_clock::now();
  const int R = planes(field);
  const int64_t wa = w64_of(l), wc = w64_of(n);
  // row pieces: Pr equal pieces, or (SG_HOST_PIECES=w0,w1,..., experiments) up to 8 pieces with
  // relative weights -- e.g. a small first piece starts the product sooner, a small last piece
  // shortens the download after the last product
  std::vector<int64_t> cuts{0};
  if (const char* e = getenv("SG_HOST_PIECES")) {
    std::vector<int64_t> w;
    for (const char* q = e; *q && w.size() < 8;) {
      w.push_back(std::max(1LL, atoll(q)));
      while (*q && *q != ',') ++q;
      if (*q == ',') ++q;
    }
    int64_t tot = 0, acc = 0;
    for (int64_t x : w) tot += x;
    for (int64_t x : w) cuts.push_back(m * (acc += x) / tot);
  } else {
    for (int r = 1; r <= Pr; ++r) cuts.push_back(m * r / Pr);
  }
  Pr = (int)cuts.size() - 1;
  auto rcut = [&](int r) { return cuts[r]; };
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
    }
    if (d->stream_ops == 0) {
      // first use of the stream memory operations while nothing waits on them; the outcome is
      // kept, so a device without them falls back on every call, not just the first
      if (wv((CUstream)d->flags, (CUdeviceptr)(d->ready + MAX_BCHUNKS), 0u, 0) != CUDA_SUCCESS ||
          cudaStreamSynchronize(d->flags) != cudaSuccess) {
        cudaGetLastError();
        d->stream_ops = -1;
        return SG_EUNSUPPORTED;
      }
      d->stream_ops = 1;
    }
  }
  unsigned* err = d->ready + MAX_BCHUNKS;
  const unsigned epoch = ++d->epoch;
  // B chunks: whole 4-block groups (32 rows): g0, then chunks of 2 g0 (chunk_lo in sg_internal.h:
  // sizes double from g0 up to g0 2^q; q = 1 by default).  The first chunk is small so the
  // product starts early; after it every chunk is small enough that the product never waits
  // long for one (B arrives at ~0.7 groups / us against ~0.5 consumed), and few enough that the
  // per-copy setup stays small.  g0 = groups / 32 by default.  F5 4096^3, in-process A/B
  // (profiles/r02bl_e2e_bcap_ab.txt): q = 1 0.687 ms, q = 2 0.697, doubling to the end
  // (q = 20, the round-1 layout whose last chunk is half of B) 0.704, q = 0 (all g0) 0.733.
  const int64_t groups = (l + 31) / 32;
  const size_t b_bytes = (size_t)R * l * wc * 8;
  const char* g0_e = getenv("SG_HOST_BFIRST");  // experiments: groups in the first chunk
  int64_t g0 = g0_e ? atoll(g0_e) : (groups + 31) / 32;
  g0 = std::max<int64_t>(1, std::min<int64_t>(g0, groups));
  // SG_HOST_BCAP=q (experiments): chunks stop doubling at g0 2^q groups
  const char* cap_e = getenv("SG_HOST_BCAP");
  const int q = cap_e ? std::max(0, std::min(20, atoi(cap_e))) : 1;
  auto chunk_lo_h = [&](int j) { return std::min<int64_t>(groups, sg::chunk_lo(j, (int)g0, q)); };
  int nch = 1;
  while (chunk_lo_h(nch) < groups) ++nch;
  if (nch > MAX_BCHUNKS) return SG_EUNSUPPORTED;
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  char* cur = dbuf;
  uint64_t* dB = (uint64_t*)cur;
  cur += up(b_bytes);
  uint64_t* dAp[8];
  for (int r = 0; r < Pr; ++r) {
    dAp[r] = (uint64_t*)cur;
    cur += up((size_t)R * (rcut(r + 1) - rcut(r)) * wa * 8);
  }
  uint64_t* dC = (uint64_t*)cur;  // pieces back to back, each [R][rows][wc]
  // SG_HOST_TRACE=1 (experiments): event timestamps of the pipeline steps on stderr
  const bool trace = getenv("SG_HOST_TRACE") != nullptr;  // read per call (experiments)
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
  // SG_HOST_DROP_FLAG=j (tests only): never publish chunk j, so the streamed product must give up
  // after its 10 s wait limit and the call must fail cleanly instead of hanging the GPU
  const char* drop_e = getenv("SG_HOST_DROP_FLAG");
  const int drop_flag = drop_e ? atoi(drop_e) : -1;
  int rc;
  // Every upload is queued before the first product: with pageable host buffers a copy call may
  // block the host until the stream's earlier work is done, and piece 0's product must never be
  // waiting for chunk flags that are not queued yet.  Order: A's piece 0, B chunk by chunk (each
  // followed by its flag), A's other pieces.
  if ((rc = upload_a(0)) != SG_OK) return rc;
  const auto t_first = std::chrono::steady_clock::now();
  for (int j = 0; j < nch; ++j) {
    const int64_t r0 = chunk_lo_h(j) * 32, rows = std::min<int64_t>(l, chunk_lo_h(j + 1) * 32) - r0;
    // Each flag goes out on its own stream behind its copy's event.  (Measured on B200: B's
    // chunks still arrive at ~30 GB/s against ~50 GB/s for one large copy -- every chunk pays
    // the copy setup; alternating two upload streams made the arrival order worse.)
    cudaStream_t cs = d->in;
    SG_CUDA(cudaMemcpy2DAsync(dB + r0 * wc, l * wc * 8, B + r0 * wc, l * wc * 8, rows * wc * 8, R,
                              cudaMemcpyHostToDevice, cs),
            "sg_m4rm_host H2D B");
    SG_CUDA(cudaEventRecord(d->ev_chunk[j], cs), "sg_m4rm_host event");
    SG_CUDA(cudaStreamWaitEvent(d->flags, d->ev_chunk[j], 0), "sg_m4rm_host wait");
    if (j == drop_flag) continue;  // test hook: a chunk that is never published
    if (wv((CUstream)d->flags, (CUdeviceptr)(d->ready + j), epoch, 0) != CUDA_SUCCESS)
      return fail(SG_ECUDA, "sg_m4rm_host: cuStreamWriteValue32 failed");
    mark("in: B chunk " + std::to_string(j) + " up", d->in);
  }
  for (int r = 1; r < Pr; ++r)
    if ((rc = upload_a(r)) != SG_OK) return rc;
  const char* poll_e = getenv("SG_HOST_POLL_NS");  // experiments: flag polling interval
  const StreamIn sin{d->ready, epoch, (int)g0, q, nch, poll_e ? (unsigned)atoi(poll_e) : 100u, err};
  // SG_HOST_STREAM=2 (experiments): the streamed kernel on fully uploaded inputs (its cost
  // without any waiting, in a warm L2)
  if (const char* e = getenv("SG_HOST_STREAM"))
    if (atoi(e) == 2) {
      SG_CUDA(cudaStreamSynchronize(d->in), "sg_m4rm_host sync");
      SG_CUDA(cudaStreamSynchronize(d->flags), "sg_m4rm_host sync");
    }
  for (int r = 0; r < Pr; ++r)
    if ((rc = product(r, r == 0 ? &sin : nullptr)) != SG_OK) return rc;
  SG_CUDA(cudaMemcpyAsync(d->err_host, err, sizeof(unsigned), cudaMemcpyDeviceToHost, d->comp), "sg_m4rm_host");
  const auto t_queued = std::chrono::steady_clock::now();
  SG_CUDA(cudaStreamSynchronize(d->out), "sg_m4rm_host sync");
  SG_CUDA(cudaStreamSynchronize(d->comp), "sg_m4rm_host sync");
  SG_CUDA(cudaStreamSynchronize(d->in), "sg_m4rm_host sync");
  SG_CUDA(cudaStreamSynchronize(d->flags), "sg_m4rm_host sync");
  if (trace) {
    auto us = [&](std::chrono::steady_clock::time_point t) {
      return std::chrono::duration<double, std::micro>(t - t_entry).count();
    };
    fprintf(stderr, "host_streamed trace Pr=%d nch=%d (host: first copy queued %.1f us, all queued %.1f us, "
            "synced %.1f us after entry)\n", Pr, nch, us(t_first), us(t_queued), us(std::chrono::steady_clock::now()));
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
}  // namespace api
}  // namespace sg

using namespace sg;
using namespace sg::api;

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
  // the pipeline proper; on failure, the copies it already queued are waited for before returning
  auto pipeline = [&]() -> int {
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
      for (auto& g : d->graphs) cudaGraphExecDestroy(g.second);  // they captured the old buffer
      d->graphs.clear();
      d->graph_seen.clear();
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
  // (an explicit SG_HOST_CHUNKS / SG_HOST_KCHUNKS request, experiments and tests, runs the pipelines)
  if (Pk == 1 && Pr == 1 && Pc == 1 && !getenv("SG_HOST_NOSMALL") && !getenv("SG_HOST_CHUNKS") &&
      !getenv("SG_HOST_KCHUNKS")) {
    // a small product (C < 1 MB, inputs < 24 MB): nothing to overlap, so everything goes on one
    // stream -- two contiguous uploads, the product, one download, one synchronization (no
    // cross-stream events: each costs a few microseconds, a large share of a ~50 us call)
    char* q = dbuf;
    uint64_t* dA = (uint64_t*)q;
    q += up(a_bytes);
    uint64_t* dB = (uint64_t*)q;
    q += up(b_bytes);
    uint64_t* dC = (uint64_t*)q;
    cudaStream_t st = d->comp;
    auto enqueue = [&]() -> int {
      if (a_bytes) SG_CUDA(cudaMemcpyAsync(dA, A, a_bytes, cudaMemcpyHostToDevice, st), "sg_m4rm_host H2D A");
      if (b_bytes) SG_CUDA(cudaMemcpyAsync(dB, B, b_bytes, cudaMemcpyHostToDevice, st), "sg_m4rm_host H2D B");
      int r = sg_m4rm(field, dA, dB, dC, m, l, n, k, nullptr, 0, st);
      if (r != SG_OK) return r;
      SG_CUDA(cudaMemcpyAsync(C, dC, c_bytes, cudaMemcpyDeviceToHost, st), "sg_m4rm_host D2H C");
      return SG_OK;
    };
    // graph replay of a repeated call: page-locked host buffers only (a pageable copy is staged
    // by the driver at call time), not under per-launch timing (experiments), SG_HOST_GRAPH=0 off
    cudaPointerAttributes pa, pb, pc;
    const bool pinned = cudaPointerGetAttributes(&pa, A) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                        cudaPointerGetAttributes(&pb, B) == cudaSuccess && pb.type == cudaMemoryTypeHost &&
                        cudaPointerGetAttributes(&pc, C) == cudaSuccess && pc.type == cudaMemoryTypeHost;
    cudaGetLastError();
    static const bool graphs_on = [] {
      const char* e = getenv("SG_HOST_GRAPH");
      return !e || atoi(e) != 0;
    }();
    if (!pinned || !graphs_on || g_timing) {
      if ((rc = enqueue()) != SG_OK) return rc;
      SG_CUDA(cudaStreamSynchronize(st), "sg_m4rm_host sync");
      return SG_OK;
    }
    Io::GraphKey key;
    {
      std::lock_guard<std::mutex> lk(g_mu);  // the plan depends on the overrides and the SM reserve
      key = Io::GraphKey{field, A, B, C, m, l, n, k,
                         {g_override_rt, g_override_splits, g_override_pipe, g_override_threads, g_ablation,
                          g_sm_reserve}};
    }
    if (d->graph_generation != g_buffer_generation.load()) {
      // a workspace or counter buffer the graphs point into was reallocated since: drop them all
      for (auto& g : d->graphs) cudaGraphExecDestroy(g.second);
      d->graphs.clear();
      d->graph_seen.clear();
      d->graph_generation = g_buffer_generation.load();
    }
    auto it = d->graphs.find(key);
    if (it == d->graphs.end()) {
      if (d->graph_seen[key]++ == 0) {  // first call: uncaptured (plans, workspaces, counters)
        if ((rc = enqueue()) != SG_OK) return rc;
        SG_CUDA(cudaStreamSynchronize(st), "sg_m4rm_host sync");
        return SG_OK;
      }
      cudaGraphExec_t ex = nullptr;
      if (d->graph_seen[key] == 2) {  // second call: capture (once; a failed capture is not retried)
        cudaGraph_t g = nullptr;
        if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
          const int r = enqueue();
          const cudaError_t ce = cudaStreamEndCapture(st, &g);
          if (r != SG_OK || ce != cudaSuccess || cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) ex = nullptr;
          if (g) cudaGraphDestroy(g);
        }
        cudaGetLastError();
      }
      if (!ex) {  // no graph for this call: the plain one-stream path
        if ((rc = enqueue()) != SG_OK) return rc;
        SG_CUDA(cudaStreamSynchronize(st), "sg_m4rm_host sync");
        return SG_OK;
      }
      if (d->graphs.size() >= 64) {
        for (auto& x : d->graphs) cudaGraphExecDestroy(x.second);
        d->graphs.clear();
      }
      it = d->graphs.emplace(key, ex).first;
    }
    SG_CUDA(cudaGraphLaunch(it->second, st), "sg_m4rm_host graph launch");
    SG_CUDA(cudaStreamSynchronize(st), "sg_m4rm_host sync");
    return SG_OK;
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
  const bool trace = getenv("SG_HOST_TRACE") != nullptr;  // read per call (experiments)
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
  };
  rc = pipeline();
  if (rc != SG_OK) drain(d);
  return rc;
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
  const size_t a_bytes = (size_t)R * m * wa * 8, b_bytes = (size_t)R * l * wc * 8, c_bytes = (size_t)R * m * wc * 8;
  // B travels in NBC row chunks (whole 64-bit words of rows) so the tree's hops pipeline
  constexpr int NBC = 8;
  struct Dev {
    cudaStream_t st = nullptr;   // A up, products, C down
    cudaStream_t cst = nullptr;  // B chunks arriving on this device (H2D or peer copy)
    cudaEvent_t ev_b[NBC];       // chunk c of B is on this device
    cudaEvent_t ev_all = nullptr;
    Buf buf;
  };
  static std::map<int, Dev> state;
  static std::mutex multi_mu;
  std::lock_guard<std::mutex> busy(multi_mu);  // one multi-device product at a time
  // distinct devices in order of first appearance; devices[0] receives B from the host
  std::vector<int> uniq;
  for (int g = 0; g < ngpus; ++g)
    if (std::find(uniq.begin(), uniq.end(), devices[g]) == uniq.end()) uniq.push_back(devices[g]);
  std::map<int, size_t> need;
  std::vector<int64_t> r0(ngpus), r1(ngpus);
  for (int g = 0; g < ngpus; ++g) {
    r0[g] = m * g / ngpus;
    r1[g] = m * (g + 1) / ngpus;
    need[devices[g]] += ((size_t)R * (r1[g] - r0[g]) * (wa + wc) * 8 + 2 * 256);
  }
  for (int dv : uniq) {
    size_t& bytes = need[dv];
    bytes += b_bytes + 256;
    Dev& d = state[dv];
    SG_CUDA(cudaSetDevice(dv), "sg_m4rm_multi set device");
    if (!d.st) {
      SG_CUDA(cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking), "sg_m4rm_multi stream");
      SG_CUDA(cudaStreamCreateWithFlags(&d.cst, cudaStreamNonBlocking), "sg_m4rm_multi stream");
      for (int c = 0; c < NBC; ++c)
        SG_CUDA(cudaEventCreateWithFlags(&d.ev_b[c], cudaEventDisableTiming), "sg_m4rm_multi event");
      SG_CUDA(cudaEventCreateWithFlags(&d.ev_all, cudaEventDisableTiming), "sg_m4rm_multi event");
    }
    if (d.buf.bytes < bytes) {
      if (d.buf.p) {
        cudaDeviceSynchronize();
        cudaFree(d.buf.p);
      }
      d.buf.p = nullptr;
      d.buf.bytes = 0;
      SG_CUDA(cudaMalloc(&d.buf.p, bytes), "sg_m4rm_multi alloc");
      d.buf.bytes = bytes;
    }
  }
  // Host buffers: page-locked for the duration of the call unless they already are, so every
  // copy is asynchronous and the devices run concurrently (a copy from or to pageable memory
  // would make the host wait for each device in turn).
  std::vector<void*> registered;
  auto pin = [&](const void* p, size_t bytes) -> int {
    if (!bytes) return SG_OK;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost) return SG_OK;
    cudaGetLastError();
    const cudaError_t e = cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterPortable);
    if (e == cudaSuccess) registered.push_back(const_cast<void*>(p));
    else cudaGetLastError();  // e.g. already registered by the caller: the copies still work
    return SG_OK;
  };
  auto finish = [&](int code) {
    for (int dv : uniq) {  // never return while a queued copy may still touch the caller's buffers
      cudaSetDevice(dv);
      cudaStreamSynchronize(state[dv].cst);
      cudaStreamSynchronize(state[dv].st);
    }
    for (void* p : registered) cudaHostUnregister(p);
    cudaGetLastError();
    cudaSetDevice(cur);
    return code;
  };
  pin(A, a_bytes);
  pin(B, b_bytes);
  pin(C, c_bytes);
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  // B: host -> uniq[0] in NBC row chunks, then a doubling tree of peer copies over NVLink /
  // NVSwitch -- in round t, device i < 2^t sends to device i + 2^t -- pipelined by chunk: chunk
  // c's hop to device j waits only for chunk c on its sender (ev_b), so hops of different chunks
  // and rounds overlap.  Every device receives B once, ceil(log2 G) hops deep, instead of G-1
  // copies leaving one device.
  const int G = (int)uniq.size();
  const int64_t bw = wc;  // words per B row
  auto brow = [&](int c) { return std::min<int64_t>(l, ((wa * c / NBC) * 64)); };  // chunk c = rows [brow(c), brow(c+1))
  auto copy_chunk = [&](int dst, int src, int c) -> int {
    const int64_t q0 = c == 0 ? 0 : brow(c), q1 = c == NBC - 1 ? l : brow(c + 1);
    Dev& d = state[uniq[dst]];
    SG_CUDA(cudaSetDevice(uniq[dst]), "sg_m4rm_multi set device");
    if (q1 > q0) {
      // R planes, rows [q0, q1) of each: one 2-D copy (pitch = a plane's bytes)
      char* dbase = (char*)d.buf.p;
      if (src < 0) {
        SG_CUDA(cudaMemcpy2DAsync(dbase + q0 * bw * 8, l * bw * 8, (const char*)B + q0 * bw * 8, l * bw * 8,
                                  (q1 - q0) * bw * 8, R, cudaMemcpyHostToDevice, d.cst),
                "sg_m4rm_multi H2D B");
      } else {
        Dev& s = state[uniq[src]];
        SG_CUDA(cudaStreamWaitEvent(d.cst, s.ev_b[c], 0), "sg_m4rm_multi wait");
        for (int p = 0; p < R; ++p)
          SG_CUDA(cudaMemcpyPeerAsync(dbase + ((int64_t)p * l + q0) * bw * 8, uniq[dst],
                                      (char*)s.buf.p + ((int64_t)p * l + q0) * bw * 8, uniq[src],
                                      (q1 - q0) * bw * 8, d.cst),
                  "sg_m4rm_multi peer copy B");
      }
    }
    SG_CUDA(cudaEventRecord(d.ev_b[c], d.cst), "sg_m4rm_multi event");
    return SG_OK;
  };
  for (int i = 1; i < G; ++i) {  // peer access for every tree edge (sender (i - 2^t) -> i)
    int hb = 1;
    while (hb * 2 <= i) hb *= 2;
    const int from = uniq[i - hb];
    SG_CUDA(cudaSetDevice(uniq[i]), "sg_m4rm_multi set device");
    int can = 0;
    cudaDeviceCanAccessPeer(&can, uniq[i], from);
    if (can) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(from, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return finish(cuda_fail(e, "sg_m4rm_multi peer access"));
      cudaGetLastError();
    }
  }
  if (b_bytes) {
    for (int c = 0; c < NBC; ++c) {
      if ((rc = copy_chunk(0, -1, c)) != SG_OK) return finish(rc);
      for (int span = 1; span < G; span *= 2)  // chunk c down the tree, round by round
        for (int i = 0; i < span && i + span < G; ++i)
          if ((rc = copy_chunk(i + span, i, c)) != SG_OK) return finish(rc);
    }
  }
  for (int dv : uniq) {
    Dev& d = state[dv];
    SG_CUDA(cudaSetDevice(dv), "sg_m4rm_multi set device");
    SG_CUDA(cudaEventRecord(d.ev_all, d.cst), "sg_m4rm_multi event");
  }
  // every shard's A upload and product first (all devices busy), the C downloads after
  std::map<int, size_t> offset;
  for (int dv : uniq) offset[dv] = up(b_bytes);
  std::vector<uint64_t*> dCs(ngpus, nullptr);
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
    dCs[g] = (uint64_t*)(base + offset[dv]);
    offset[dv] += up((size_t)R * rows * wc * 8);
    if (wa)
      SG_CUDA(cudaMemcpy2DAsync(dA, rows * wa * 8, A + r0[g] * wa, m * wa * 8, rows * wa * 8, R,
                                cudaMemcpyHostToDevice, d.st),
              "sg_m4rm_multi H2D A");
    SG_CUDA(cudaStreamWaitEvent(d.st, d.ev_all, 0), "sg_m4rm_multi wait");  // all of B is here
    rc = sg_m4rm(field, dA, dB, dCs[g], rows, l, n, k, nullptr, 0, d.st);
    if (rc != SG_OK) return finish(rc);
  }
  for (int g = 0; g < ngpus; ++g) {
    if (!dCs[g]) continue;
    const int64_t rows = r1[g] - r0[g];
    SG_CUDA(cudaSetDevice(devices[g]), "sg_m4rm_multi set device");
    SG_CUDA(cudaMemcpy2DAsync(C + r0[g] * wc, m * wc * 8, dCs[g], rows * wc * 8, rows * wc * 8, R,
                              cudaMemcpyDeviceToHost, state[devices[g]].st),
            "sg_m4rm_multi D2H C");
  }
  for (int dv : uniq) {
    SG_CUDA(cudaSetDevice(dv), "sg_m4rm_multi set device");
    const cudaError_t e = cudaStreamSynchronize(state[dv].st);
    if (e != cudaSuccess) return finish(cuda_fail(e, "sg_m4rm_multi sync"));
  }
  return finish(SG_OK);
}

}  // extern "C"

// multi_host.cu -- my_dgemm_multi: the host-pointer drop-in spread over
// several GPUs of one process (SURVEY.md 8b "my_dgemm_multi(int ngpu, ...)";
// the multi-process NCCL form is paper_1609_00076_b200/multi.py).
//
// Sharding follows 8e: shard s owns the contiguous column panel [j0, j1) of
// B and C (split_columns: balanced, 128-column units, multi.py), so B and C
// cross only that device's own PCIe link.  A is needed whole on every
// device; instead of every device pulling all of A over PCIe (or one root
// pulling it and then broadcasting), the k-chunks of A are uploaded
// round-robin -- chunk c by shard c mod G over shard c's PCIe link -- and
// every other shard copies it peer to peer (NVLink on a B200 box).  So each
// link carries A/G + its own B and C panels, and the chunks' peer copies
// overlap the GEMMs of earlier chunks.
//
// Each shard runs C_s += A[:, chunk] B_s[chunk, :] for chunks in ascending
// order on its own stream: chunks are multiples of 16 (the kernel's K slab),
// so the per-element DMMA sequence -- hence C -- is bitwise the
// single-device call for every device count (tests/test_gpu_parity.py).
//
// One host thread per shard issues that shard's copies and launches.  A
// thread waits (host side) for a chunk's upload to have been *recorded* by
// its owner before queueing the peer copy behind that event; chunks are
// handled in ascending order by every thread, so the chunk-c owner only ever
// waits on chunks < c: no cycle.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/my_dgemm.h"
#include "common.cuh"
#include "host_io.cuh"

namespace myd {

cudaError_t dispatch(int m, int n, int k, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                     int64_t ldc, cudaStream_t st, unsigned flags, const Epilogue &ep);
int host_path(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc,
              unsigned flags);
int path_kind(int m, int n, unsigned flags);
int capi_fail(int status, const std::string &msg);
int capi_ok();
int capi_cuda_fail(cudaError_t e, const char *where);

namespace {

constexpr int MAX_SHARDS = 64;

struct ShardWs {
  int device = -1;
  double *dA = nullptr, *dB = nullptr, *dC = nullptr;
  size_t capA = 0, capB = 0, capC = 0;
  cudaStream_t s_up = nullptr, s_peer = nullptr, s_comp = nullptr, s_down = nullptr;
  std::vector<cudaEvent_t> ev_a, ev_b;  // per chunk: A chunk resident here, B rows uploaded
  cudaEvent_t ev_done = nullptr;
  hostio::StageRing stage;

  void release() {
    if (device < 0) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (cudaStream_t s : {s_up, s_peer, s_comp, s_down})
      if (s) cudaStreamSynchronize(s);
    if (dA) cudaFree(dA);
    if (dB) cudaFree(dB);
    if (dC) cudaFree(dC);
    dA = dB = dC = nullptr;
    capA = capB = capC = 0;
    for (cudaEvent_t e : ev_a) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_b) cudaEventDestroy(e);
    ev_a.clear();
    ev_b.clear();
    if (ev_done) cudaEventDestroy(ev_done);
    ev_done = nullptr;
    for (cudaStream_t s : {s_up, s_peer, s_comp, s_down})
      if (s) cudaStreamDestroy(s);
    s_up = s_peer = s_comp = s_down = nullptr;
    stage.release();
    cudaSetDevice(prev);
    device = -1;
  }
};

std::mutex g_multi_mutex;  // one multi-device call at a time (shared shard workspaces)
ShardWs g_shards[MAX_SHARDS];

cudaError_t grow(double **p, size_t *cap, size_t need) {
  if (*cap >= need) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc((void **)p, need);
  if (e == cudaSuccess) *cap = need;
  return e;
}

// Chunks whose upload has been recorded (1), or abandoned by a failing owner (-1).
struct ChunkBoard {
  std::mutex mu;
  std::condition_variable cv;
  std::vector<int> state;
  void post(size_t c, int v) {
    {
      std::lock_guard<std::mutex> lk(mu);
      state[c] = v;
    }
    cv.notify_all();
  }
  int wait(size_t c) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return state[c] != 0; });
    return state[c];
  }
};

struct Problem {
  int m, n, k;
  const double *A;
  int lda;
  const double *B;
  int ldb;
  double *C;
  int ldc;
  unsigned flags;
  int64_t dlda, dldb, dldc;
  std::vector<std::pair<int64_t, int64_t>> cols, chunks;
  bool staged;
};

struct ShardResult {
  cudaError_t err = cudaSuccess;
  const char *where = "";
};

void run_shard(int s, int G, Problem &P, ChunkBoard &board, ShardResult &res) {
  ShardWs &w = g_shards[s];
  const size_t nch = P.chunks.size();
  std::vector<bool> posted(nch, false);
  auto fail = [&](cudaError_t e, const char *where) {
    res.err = e;
    res.where = where;
    for (size_t c = 0; c < nch; ++c)  // release anyone waiting on this shard's chunks
      if ((int)(c % G) == s && !posted[c]) board.post(c, -1);
  };
  cudaError_t e;
  if ((e = cudaSetDevice(w.device)) != cudaSuccess) return fail(e, "cudaSetDevice");
  const int64_t j0 = P.cols[s].first, nloc = P.cols[s].second - P.cols[s].first;
  if ((e = grow(&w.dA, &w.capA, (size_t)P.dlda * P.k * 8)) != cudaSuccess) return fail(e, "cudaMalloc(A)");
  if (nloc > 0) {
    if ((e = grow(&w.dB, &w.capB, (size_t)P.dldb * nloc * 8)) != cudaSuccess) return fail(e, "cudaMalloc(B)");
    if ((e = grow(&w.dC, &w.capC, (size_t)P.dldc * nloc * 8)) != cudaSuccess) return fail(e, "cudaMalloc(C)");
  }
  if (P.staged && (e = w.stage.ensure(4)) != cudaSuccess) return fail(e, "pinned staging");
  hostio::Mover mv(P.staged ? &w.stage : nullptr, w.s_up, w.s_down);
  const Epilogue ep{};
  // Every shard runs the whole problem's kernel family (a narrow panel must
  // not switch kernels: their summation orders differ).
  const unsigned flags = P.flags | MY_DGEMM_FORCE_PATH(path_kind(P.m, P.n, P.flags));

  if (nloc > 0 && (e = mv.up(w.dC, P.dldc, P.C + j0 * P.ldc, P.ldc, P.m, nloc)) != cudaSuccess)
    return fail(e, "H2D C");
  for (size_t c = 0; c < nch; ++c) {
    const int64_t p0 = P.chunks[c].first, kc = P.chunks[c].second - p0;
    const int owner = (int)(c % G);
    if (owner == s) {  // this shard's link carries chunk c of A
      if ((e = mv.up(w.dA + p0 * P.dlda, P.dlda, P.A + p0 * P.lda, P.lda, P.m, kc)) != cudaSuccess)
        return fail(e, "H2D A");
      if ((e = cudaEventRecord(w.ev_a[c], w.s_up)) != cudaSuccess) return fail(e, "cudaEventRecord");
      board.post(c, 1);
      posted[c] = true;
    }
    if (nloc > 0) {
      if ((e = mv.up(w.dB + p0, P.dldb, P.B + j0 * P.ldb + p0, P.ldb, kc, nloc)) != cudaSuccess)
        return fail(e, "H2D B");
      if ((e = cudaEventRecord(w.ev_b[c], w.s_up)) != cudaSuccess) return fail(e, "cudaEventRecord");
    }
    if (owner != s) {  // peer copy of chunk c from its owner
      if (board.wait(c) < 0) return fail(cudaErrorUnknown, "peer shard failed");
      ShardWs &o = g_shards[owner];
      if ((e = cudaStreamWaitEvent(w.s_peer, o.ev_a[c], 0)) != cudaSuccess) return fail(e, "cudaStreamWaitEvent");
      e = cudaMemcpyPeerAsync(w.dA + p0 * P.dlda, w.device, o.dA + p0 * P.dlda, o.device,
                              (size_t)((kc - 1) * P.dlda + P.m) * 8, w.s_peer);
      if (e != cudaSuccess) return fail(e, "peer copy of A");
      if ((e = cudaEventRecord(w.ev_a[c], w.s_peer)) != cudaSuccess) return fail(e, "cudaEventRecord");
    }
    if (nloc > 0) {
      cudaStreamWaitEvent(w.s_comp, w.ev_a[c], 0);
      cudaStreamWaitEvent(w.s_comp, w.ev_b[c], 0);
      e = dispatch(P.m, (int)nloc, (int)kc, w.dA + p0 * P.dlda, P.dlda, w.dB + p0, P.dldb, w.dC, P.dldc, w.s_comp,
                   flags, ep);
      if (e != cudaSuccess) return fail(e, "kernel launch");
    }
  }
  if (nloc > 0) {
    // the panel's C goes down once final and once every upload of this link is queued
    cudaEventRecord(w.ev_done, w.s_comp);
    cudaStreamWaitEvent(w.s_down, w.ev_done, 0);
    cudaStreamWaitEvent(w.s_down, w.ev_b[nch - 1], 0);
    if ((e = mv.down(P.C + j0 * P.ldc, P.ldc, w.dC, P.dldc, P.m, nloc)) != cudaSuccess) return fail(e, "D2H C");
    if ((e = mv.finish()) != cudaSuccess) return fail(e, "D2H C");
  }
  // Peers may still be reading this shard's A chunks: the caller
  // synchronises every shard's streams before returning.
}

cudaError_t prepare_shard(int s, int device, size_t nch) {
  ShardWs &w = g_shards[s];
  if (w.device != device) w.release();
  w.device = device;
  cudaError_t e;
  if ((e = cudaSetDevice(device)) != cudaSuccess) return e;
  if (!w.s_up) {
    for (cudaStream_t *p : {&w.s_up, &w.s_peer, &w.s_comp, &w.s_down})
      if ((e = cudaStreamCreateWithFlags(p, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&w.ev_done, cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  while (w.ev_a.size() < nch) {
    cudaEvent_t a, b;
    if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming)) != cudaSuccess) return e;
    w.ev_a.push_back(a);
    w.ev_b.push_back(b);
  }
  return cudaSuccess;
}

}  // namespace

// multi.py split_columns: contiguous balanced panels in 128-column units.
std::vector<std::pair<int64_t, int64_t>> split_columns(int64_t n, int parts, int64_t align = 128) {
  std::vector<std::pair<int64_t, int64_t>> out;
  const int64_t units = (n + align - 1) / align, base = units / parts, rem = units % parts;
  int64_t lo = 0;
  for (int w = 0; w < parts; ++w) {
    const int64_t hi = std::min<int64_t>(n, lo + (base + (w < rem ? 1 : 0)) * align);
    out.push_back({lo, hi});
    lo = hi;
  }
  return out;
}

int multi_host_path(const int *devices, int G, int m, int n, int k, const double *A, int lda, const double *B,
                    int ldb, double *C, int ldc, unsigned flags) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (G == 1) {
    cudaError_t e = cudaSetDevice(devices[0]);
    if (e != cudaSuccess) return capi_cuda_fail(e, "cudaSetDevice");
    const int st = host_path(m, n, k, A, lda, B, ldb, C, ldc, flags);
    cudaSetDevice(prev);
    return st;
  }
  std::lock_guard<std::mutex> lock(g_multi_mutex);
  Problem P{m, n, k, A, lda, B, ldb, C, ldc, flags, (m + 1) & ~1LL, (k + 1) & ~1LL, (m + 1) & ~1LL, {}, {}, false};
  P.cols = split_columns(n, G);
  // k-chunks (multiples of 16): about two per shard, at least 256 deep.  The
  // bandwidth kernels split k their own way (their sums are not
  // chunk-invariant): one chunk there, as the single-device call.
  const int64_t want = std::max<int64_t>(G, std::min<int64_t>(4LL * G, k / 256));
  const int64_t kchunk = path_kind(m, n, flags) != MY_DGEMM_PATH_TILED
                             ? k
                             : std::max<int64_t>(16, ((k + want - 1) / want + 15) / 16 * 16);
  for (int64_t p = 0; p < k; p += kchunk) P.chunks.push_back({p, std::min<int64_t>(k, p + kchunk)});
  P.staged = !(hostio::is_pinned(A) && hostio::is_pinned(B) && hostio::is_pinned(C));
  cudaError_t e = cudaSuccess;
  for (int s = 0; s < G && e == cudaSuccess; ++s) e = prepare_shard(s, devices[s], P.chunks.size());
  if (e != cudaSuccess) {
    cudaSetDevice(prev);
    return capi_cuda_fail(e, "multi-device setup");
  }
  // peer access between distinct devices (NVLink / PCIe P2P); the copies
  // also work without it, staged through the host by the driver
  for (int a = 0; a < G; ++a)
    for (int b = 0; b < G; ++b) {
      if (devices[a] == devices[b]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[a], devices[b]);
      if (can) {
        cudaSetDevice(devices[a]);
        cudaDeviceEnablePeerAccess(devices[b], 0);  // already enabled: harmless error
        cudaGetLastError();
      }
    }
  ChunkBoard board;
  board.state.assign(P.chunks.size(), 0);
  std::vector<ShardResult> res(G);
  std::vector<std::thread> threads;
  for (int s = 0; s < G; ++s) threads.emplace_back(run_shard, s, G, std::ref(P), std::ref(board), std::ref(res[s]));
  for (auto &t : threads) t.join();
  cudaError_t first = cudaSuccess;
  const char *where = "";
  for (int s = 0; s < G; ++s) {
    ShardWs &w = g_shards[s];
    cudaSetDevice(w.device);
    for (cudaStream_t st : {w.s_up, w.s_peer, w.s_comp, w.s_down}) {
      cudaError_t e2 = cudaStreamSynchronize(st);
      if (first == cudaSuccess && e2 != cudaSuccess) {
        first = e2;
        where = "synchronize";
      }
    }
  }
  for (int s = 0; s < G; ++s)
    if (res[s].err != cudaSuccess && res[s].err != cudaErrorUnknown) {
      first = res[s].err;
      where = res[s].where;
      break;
    }
  if (first == cudaSuccess)
    for (int s = 0; s < G; ++s)
      if (res[s].err != cudaSuccess) {
        first = res[s].err;
        where = res[s].where;
        break;
      }
  cudaSetDevice(prev);
  if (first != cudaSuccess) return capi_cuda_fail(first, where);
  return capi_ok();
}

void release_multi_workspace() {
  std::lock_guard<std::mutex> lock(g_multi_mutex);
  for (auto &w : g_shards) w.release();
}

}  // namespace myd

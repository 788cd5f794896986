// host_path.cu -- my_dgemm on HOST pointers: the drop-in CPU signature
// driving the device kernels, with the transfers pipelined
// against the GEMM.
//
// Measured on the B200 box (tools/pcie_probe.py): PCIe 5 moves 55.5 GB/s
// H2D and 56.8 GB/s D2H from pinned memory but only ~34 GB/s in total when
// both directions run at once, and 26.7 / 17.5 GB/s from pageable memory.
// Schedule (modelled by tools/e2e_schedule_sim.py):
//   * uploads first, downloads deferred until every upload is queued;
//   * the first column group (half of C) is computed in k-chunks while A is
//     still uploading (chunks are multiples of 16: bitwise the unchunked
//     result), the remaining panels run whole as their B and C land;
//   * each panel's C goes down as soon as it is final.
// Pageable callers (numpy arrays, the reference's own Matrix objects) go
// through a pinned staging ring filled and drained by a small pool of host
// threads, so the DMA engines always see pinned memory (host_io.cuh).
#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/my_dgemm.h"
#include "common.cuh"
#include "host_io.cuh"

namespace myd {

cudaError_t dispatch(int m, int n, int k, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                     int64_t ldc, cudaStream_t st, unsigned flags, const Epilogue &ep);
int path_kind(int m, int n, unsigned flags);
int capi_fail(int status, const std::string &msg);
int capi_ok();
int capi_cuda_fail(cudaError_t e, const char *where);

namespace {

struct Workspace {
  int device = -1;
  double *dA = nullptr, *dB = nullptr, *dC = nullptr;
  size_t capA = 0, capB = 0, capC = 0;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_done, ev_out;
  hostio::StageRing stage;  // pinned staging ring for pageable callers
};

std::mutex g_ws_mutex;
Workspace g_ws[64];

cudaError_t grow(double **p, size_t *cap, size_t need) {
  if (*cap >= need) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc((void **)p, need);
  if (e == cudaSuccess) *cap = need;
  return e;
}

cudaError_t ensure_streams(Workspace &w, size_t n_events) {
  cudaError_t e;
  if (!w.s_h2d) {
    if ((e = cudaStreamCreateWithFlags(&w.s_h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&w.s_comp, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&w.s_d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
  }
  while (w.ev_in.size() < n_events) {
    cudaEvent_t a, b, c;
    if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&c, cudaEventDisableTiming)) != cudaSuccess) return e;
    w.ev_in.push_back(a);
    w.ev_done.push_back(b);
    w.ev_out.push_back(c);
  }
  return cudaSuccess;
}


}  // namespace

int host_path(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc,
              unsigned flags) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return capi_cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return capi_fail(-11, "device index out of range");
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  Workspace &w = g_ws[dev];
  w.device = dev;
  // Device copies use even leading dimensions so every column starts 16-byte
  // aligned and the bulk-copy staging path applies whatever the host ld was.
  const int64_t dlda = (m + 1) & ~1LL, dldb = (k + 1) & ~1LL, dldc = (m + 1) & ~1LL;
  const double flops = 2.0 * m * (double)n * k;
  // (the column panels and k-chunks are bitwise the one call only on the tiled path)
  const bool pipelined = flops > 4e9 && n >= 1024 && path_kind(m, n, flags) == MY_DGEMM_PATH_TILED;
  // (its panels and k-chunks must each keep the one call's arithmetic: plan-invariant plans only)
  if (pipelined) flags |= MY_DGEMM_PLAN_INVARIANT;
  // Column group 0 is computed in k-chunks while A uploads; it only needs to
  // be wide enough that each chunk's GEMM outlasts the next chunk's upload
  // (flop per uploaded byte 2 m nc0 / (8 (m + nc0)) against 36.7 TF over
  // 55 GB/s, with 25 % margin), and no wider: its C block is the upload the
  // first GEMM waits for.  Small m cannot hide A at all; then half of C.
  // The remaining columns go in panels of ~n/8 whose last one is cut into
  // halves down to 512 columns, so the download after the final GEMM is short.
  int64_t nc0 = n;
  std::vector<int64_t> pj0, pnc;  // panels after group 0: first column, width
  if (pipelined) {
    const double need = 1.25 * 8.0 * 36.7e12 / (2.0 * 55e9);  // m nc0 / (m + nc0) >= need
    nc0 = std::max<int64_t>(128, (n / 2) / 128 * 128);
    if ((double)m > need * 1.05) {
      const double w = need * m / (m - need);
      nc0 = std::min<int64_t>(nc0, std::max<int64_t>(1024, ((int64_t)w + 127) / 128 * 128));
    }
    const int64_t panel = std::max<int64_t>(512, ((n / 8 + 127) / 128) * 128);
    for (int64_t j = nc0; j < n;) {
      int64_t wdt = std::min<int64_t>(panel, n - j);
      pj0.push_back(j);
      pnc.push_back(wdt);
      j += wdt;
    }
    while (!pnc.empty() && pnc.back() >= 1024) {  // halve the last panel: 4096 -> 2048, 1024, 512, 512
      const int64_t last = pnc.back(), h = (last / 2 + 127) / 128 * 128;
      if (last - h < 512) break;
      pnc.back() = h;
      pj0.push_back(pj0.back() + h);
      pnc.push_back(last - h);
      if (last - h < 1024) break;
    }
  }
  const size_t panels = 1 + pj0.size();  // group 0 + whole panels
  auto panel_j0 = [&](size_t p) -> int64_t { return p == 0 ? 0 : pj0[p - 1]; };
  auto panel_nc = [&](size_t p) -> int64_t { return p == 0 ? nc0 : pnc[p - 1]; };
  int64_t kchunk = k;  // multiples of 16: bitwise the unchunked GEMM
  if (pipelined && k >= 256) kchunk = std::min<int64_t>(1024, (((k + 7) / 8) + 15) / 16 * 16);
  const size_t kchunks = (size_t)((k + kchunk - 1) / kchunk);
  if ((e = ensure_streams(w, std::max(panels, kchunks) + 1)) != cudaSuccess)
    return capi_cuda_fail(e, "stream setup");
  if ((e = grow(&w.dA, &w.capA, (size_t)dlda * k * 8)) != cudaSuccess) return capi_cuda_fail(e, "cudaMalloc(A)");
  if ((e = grow(&w.dB, &w.capB, (size_t)dldb * n * 8)) != cudaSuccess) return capi_cuda_fail(e, "cudaMalloc(B)");
  if ((e = grow(&w.dC, &w.capC, (size_t)dldc * n * 8)) != cudaSuccess) return capi_cuda_fail(e, "cudaMalloc(C)");
  const bool staged = !(hostio::is_pinned(A) && hostio::is_pinned(B) && hostio::is_pinned(C));
  if (staged && (e = w.stage.ensure(6)) != cudaSuccess) return capi_cuda_fail(e, "pinned staging");
  hostio::Mover mv(staged ? &w.stage : nullptr, w.s_h2d, w.s_d2h);
  const Epilogue ep{};

  // Program order = issue order: every GEMM is queued right after the
  // uploads it needs, so the device never waits for the host to finish
  // staging unrelated data.
  // The first k-chunk of group 0 runs in column pieces, each as soon as its
  // C and B land after A's first chunk, so the first GEMM waits for ~1/4 of
  // group 0's C instead of all of it (column pieces: bitwise the one call).
  size_t c_first = 0;
  if (pipelined && kchunks > 1 && nc0 >= 1024) {
    const int64_t kl = kchunk, piece = ((nc0 / 4) + 127) / 128 * 128;
    if ((e = mv.up(w.dA, dlda, A, lda, m, kl)) != cudaSuccess) return capi_cuda_fail(e, "H2D A");
    for (int64_t j0 = 0; j0 < nc0; j0 += piece) {
      const int64_t nc = std::min<int64_t>(piece, nc0 - j0);
      if ((e = mv.up(w.dC + j0 * dldc, dldc, C + j0 * ldc, ldc, m, nc)) != cudaSuccess)
        return capi_cuda_fail(e, "H2D C");
      if ((e = mv.up(w.dB + j0 * dldb, dldb, B + j0 * ldb, ldb, kl, nc)) != cudaSuccess)
        return capi_cuda_fail(e, "H2D B");
      cudaEventRecord(w.ev_in[0], w.s_h2d);  // (each wait takes the record before it)
      cudaStreamWaitEvent(w.s_comp, w.ev_in[0], 0);
      e = dispatch(m, (int)nc, (int)kl, w.dA, dlda, w.dB + j0 * dldb, dldb, w.dC + j0 * dldc, dldc, w.s_comp, flags,
                   ep);
      if (e != cudaSuccess) return capi_cuda_fail(e, "kernel launch");
    }
    c_first = 1;
  } else if ((e = mv.up(w.dC, dldc, C, ldc, m, nc0)) != cudaSuccess) {
    return capi_cuda_fail(e, "H2D C");
  }
  for (size_t c = c_first; c < kchunks; ++c) {  // group 0: k-chunks as A arrives
    const int64_t p0 = (int64_t)c * kchunk, kl = std::min<int64_t>(kchunk, k - p0);
    if ((e = mv.up(w.dA + p0 * dlda, dlda, A + p0 * lda, lda, m, kl)) != cudaSuccess)
      return capi_cuda_fail(e, "H2D A");
    if ((e = mv.up(w.dB + p0, dldb, B + p0, ldb, kl, nc0)) != cudaSuccess) return capi_cuda_fail(e, "H2D B");
    cudaEventRecord(w.ev_in[c], w.s_h2d);
    cudaStreamWaitEvent(w.s_comp, w.ev_in[c], 0);
    e = dispatch(m, (int)nc0, (int)kl, w.dA + p0 * dlda, dlda, w.dB + p0, dldb, w.dC, dldc, w.s_comp, flags, ep);
    if (e != cudaSuccess) return capi_cuda_fail(e, "kernel launch");
  }
  cudaEventRecord(w.ev_out[0], w.s_comp);
  for (size_t p = 1; p < panels; ++p) {  // whole panels as their B and C land
    const int64_t j0 = panel_j0(p), nc = panel_nc(p);
    if ((e = mv.up(w.dB + j0 * dldb, dldb, B + j0 * ldb, ldb, k, nc)) != cudaSuccess)
      return capi_cuda_fail(e, "H2D B");
    if ((e = mv.up(w.dC + j0 * dldc, dldc, C + j0 * ldc, ldc, m, nc)) != cudaSuccess)
      return capi_cuda_fail(e, "H2D C");
    cudaEventRecord(w.ev_done[p], w.s_h2d);
    cudaStreamWaitEvent(w.s_comp, w.ev_done[p], 0);
    e = dispatch(m, (int)nc, k, w.dA, dlda, w.dB + j0 * dldb, dldb, w.dC + j0 * dldc, dldc, w.s_comp, flags, ep);
    if (e != cudaSuccess) return capi_cuda_fail(e, "kernel launch");
    cudaEventRecord(w.ev_out[p], w.s_comp);
  }
  cudaEvent_t all_in = w.ev_in[kchunks];  // every upload done: downloads may start
  cudaEventRecord(all_in, w.s_h2d);
  cudaStreamWaitEvent(w.s_d2h, all_in, 0);
  for (size_t p = 0; p < panels; ++p) {
    const int64_t j0 = panel_j0(p), nc = panel_nc(p);
    cudaStreamWaitEvent(w.s_d2h, w.ev_out[p], 0);
    if ((e = mv.down(C + j0 * ldc, ldc, w.dC + j0 * dldc, dldc, m, nc)) != cudaSuccess)
      return capi_cuda_fail(e, "D2H C");
  }
  if ((e = mv.finish()) != cudaSuccess) return capi_cuda_fail(e, "D2H C");
  if ((e = cudaStreamSynchronize(w.s_d2h)) != cudaSuccess) return capi_cuda_fail(e, "synchronize");
  if ((e = cudaStreamSynchronize(w.s_comp)) != cudaSuccess) return capi_cuda_fail(e, "synchronize");
  return capi_ok();
}

void release_host_workspace() {
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  for (auto &w : g_ws) {
    if (w.device < 0) continue;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(w.device);
    if (w.dA) cudaFree(w.dA);
    if (w.dB) cudaFree(w.dB);
    if (w.dC) cudaFree(w.dC);
    w.dA = w.dB = w.dC = nullptr;
    w.capA = w.capB = w.capC = 0;
    w.stage.release();
    cudaSetDevice(prev);
  }
}

}  // namespace myd

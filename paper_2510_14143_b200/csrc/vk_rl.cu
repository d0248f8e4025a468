// C-ABI implementation of include/vk_rl.h: plans, device buffers, the RL
// iteration driver and the reference's validation / stopping semantics.
//
// Reference behaviour mirrored here (paths relative to /root/reference/proj):
//   validation order + messages ........ src/deconv.cpp:306-326
//   padded domain / FFT grid ............ src/deconv.cpp:114-116, 205-219
//   PSF spectra (plain + flipped) ....... src/deconv.cpp:110-131
//   iteration loop / trace / stopping ... src/deconv.cpp:346-430, 296-300
//   si_psnr ............................. src/metrics.cpp:67-101
//   good_size ........................... src/fft_plan.cpp:41-49
#include <cuda_runtime.h>
#include <unistd.h>  // environ
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <list>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vk_rl.h"
#include "fast_table.h"
#include "rl_passes.cuh"
#include "rl_metrics.cuh"

using vk::Geom;
using vk::LinePlan;

namespace {

thread_local std::string g_last_error;

struct Fail {
  vk_status code;
  std::string msg;
};

[[noreturn]] void fail(vk_status code, std::string msg) { throw Fail{code, std::move(msg)}; }

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) fail(VK_ERR_OOM, std::string("device allocation failed: ") + what);
  fail(VK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
vk_status guarded(F&& f) {
  try {
    f();
    return VK_OK;
  } catch (const Fail& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return VK_ERR_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return VK_ERR_ARG;
  }
}

}  // namespace

// Shared with the other C-ABI translation units (vk_io.cpp, vk_synth.cu).
namespace vk {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace vk

namespace {

uint64_t good_size(uint64_t n) {
  if (n <= 1) return 1;
  for (uint64_t c = n;; ++c) {
    uint64_t m = c;
    for (uint64_t p : {2ull, 3ull, 5ull})
      while (m % p == 0) m /= p;
    if (m == 1) return c;
  }
}

// ---- guard bands (VK_RL_GUARD=1) --------------------------------------------
// compute-sanitizer is closed on the GPU pool this was built on, so plan
// buffers can carry their own out-of-bounds-write check: every device
// allocation gets a 64 KB band of a fixed byte pattern on each side; the bands
// are verified when the buffer is freed and by vk_debug_guard_check().
constexpr size_t kGuard = 64 << 10;
constexpr unsigned char kGuardByte = 0xA5;
bool guard_on() {
  static const bool on = [] {
    const char* e = std::getenv("VK_RL_GUARD");
    return e && e[0] == '1';
  }();
  return on;
}
struct GuardReg {
  std::mutex mu;
  std::vector<std::pair<char*, std::pair<size_t, std::string>>> live;  // raw base, (payload bytes, name)
  long long violations = 0;
  static GuardReg& get() {
    static GuardReg* g = new GuardReg();
    return *g;
  }
  // 1 if either band of `raw` no longer holds the pattern
  static int damaged(char* raw, size_t bytes, const std::string& what) {
    std::vector<unsigned char> h(kGuard);
    for (int side = 0; side < 2; ++side) {
      char* band = side ? raw + kGuard + bytes : raw;
      if (cudaMemcpy(h.data(), band, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
      for (size_t i = 0; i < kGuard; ++i)
        if (h[i] != kGuardByte) {
          std::fprintf(stderr, "vk guard: %s band of '%s' (%zu bytes) overwritten at byte %zu\n",
                       side ? "upper" : "lower", what.c_str(), bytes, side ? i : kGuard - i);
          return 1;
        }
    }
    return 0;
  }
};

// RAII device pointer owned by a plan.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count, const char* what) {
    free();
    if (count == 0) count = 1;
    if (guard_on()) {
      char* raw = nullptr;
      const size_t bytes = count * sizeof(T);
      ck(cudaMalloc(&raw, bytes + 2 * kGuard), what);
      ck(cudaMemset(raw, kGuardByte, kGuard), what);
      ck(cudaMemset(raw + kGuard + bytes, kGuardByte, kGuard), what);
      p = reinterpret_cast<T*>(raw + kGuard);
      GuardReg& g = GuardReg::get();
      std::lock_guard<std::mutex> lk(g.mu);
      g.live.push_back({raw, {bytes, what}});
    } else {
      ck(cudaMalloc(&p, count * sizeof(T)), what);
    }
    n = count;
  }
  void free() {
    if (p && guard_on()) {
      char* raw = reinterpret_cast<char*>(p) - kGuard;
      GuardReg& g = GuardReg::get();
      std::lock_guard<std::mutex> lk(g.mu);
      for (size_t i = 0; i < g.live.size(); ++i)
        if (g.live[i].first == raw) {
          cudaDeviceSynchronize();
          g.violations += GuardReg::damaged(raw, g.live[i].second.first, g.live[i].second.second);
          g.live.erase(g.live.begin() + i);
          break;
        }
      cudaFree(raw);
    } else if (p) {
      cudaFree(p);
    }
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { free(); }
};

// Radix schedule: as many radix-8 stages as the power of two allows (4,4 for
// a remainder of 2^4), then 5s and 3s.
LinePlan make_line_plan(int n, const float2* tw) {
  LinePlan p{};
  p.n = n;
  p.tw = tw;
  int m = n, e2 = 0;
  while (m % 2 == 0) {
    m /= 2;
    ++e2;
  }
  std::vector<int> r;
  while (e2 > 0) {
    if (e2 == 4) {
      r.push_back(4);
      r.push_back(4);
      e2 = 0;
    } else if (e2 >= 3) {
      r.push_back(8);
      e2 -= 3;
    } else if (e2 == 2) {
      r.push_back(4);
      e2 = 0;
    } else {
      r.push_back(2);
      e2 = 0;
    }
  }
  while (m % 5 == 0) {
    r.push_back(5);
    m /= 5;
  }
  while (m % 3 == 0) {
    r.push_back(3);
    m /= 3;
  }
  if (m != 1) fail(VK_ERR_ARG, "FFT length " + std::to_string(n) + " is not 5-smooth");
  if ((int)r.size() > vk::kMaxStages) fail(VK_ERR_ARG, "FFT length too large");
  int ns = 1;
  p.nst = (int)r.size();
  for (int s = 0; s < p.nst; ++s) {
    p.rad[s] = r[s];
    p.ns[s] = ns;
    ns *= r[s];
  }
  return p;
}

std::vector<float2> twiddles(int n) {
  std::vector<float2> t(n);
  for (int m = 0; m < n; ++m) {
    const double a = -2.0 * M_PI * (double)m / (double)n;
    t[m] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  return t;
}

// Butterfly-major pass-2 twiddles of a fast length (reg::load_twiddles2
// layout) from its natural table tw[m] = w_N^m.
std::vector<float2> fast_twiddles(const vk::FastEntry* e, const std::vector<float2>& tw) {
  const int R1 = e->R1, R2 = e->N / R1;
  std::vector<float2> t((size_t)R1 * R2);
  for (int j = 0; j < R1; ++j)
    for (int r = 0; r < R2; ++r) t[(size_t)j * R2 + r] = tw[(size_t)r * j];
  return t;
}

// Largest power-of-two line count (<= lmax) whose ping-pong smem fits `cap`.
int pick_lines(int n, int lmax, size_t cap, size_t (*bytes)(int n, int L)) {
  int L = lmax;
  while (L > 1 && bytes(n, L) > cap) L >>= 1;
  return L;
}
size_t x_smem(int Wx, int L) {
  const size_t LP = vk::line_pitch(L), Hx = Wx / 2 + 1;
  return (Wx * LP + std::max<size_t>(Wx * LP, 2 * L * Hx)) * sizeof(float2);
}
size_t yz_smem(int N, int L) { return 2 * (size_t)N * vk::line_pitch(L) * sizeof(float2); }

// VK_RL_TIMING=1: host-side phase times of the host-buffer calls on stderr
bool timing_on() {
  static const bool on = [] {
    const char* e = std::getenv("VK_RL_TIMING");
    return e && e[0] == '1';
  }();
  return on;
}

// ---- host staging -----------------------------------------------------------
// Host-pointer calls (vk_rl_run, vk_rl_step, vk_conv_run, the batch form)
// take whatever memory the caller has: pinned pointers are DMA'd directly;
// pageable ones go through a per-plan ring of pinned chunks.  The host copy of
// chunk c+1 (split over a process-wide worker pool) overlaps the DMA of chunk
// c, so a pageable call costs about max(PCIe, host memcpy) instead of both.

// Process-wide workers for parallel host memcpy.  run(n, f) calls f(0..n-1)
// on the pool and the calling thread and returns when all are done; the tasks
// never block, so concurrent callers (batch lanes) cannot deadlock.
// Staging calls it once per chunk, back to back, so dispatch latency matters:
// idle workers spin for a while before they sleep on the condition variable,
// the caller helps drain the queue, and completion is a spin on an atomic
// count (a condition-variable round trip per chunk cost ~0.15 ms:
// profiles/r02/staging_dma.md).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();  // process lifetime
    return *p;
  }
  int size() const { return (int)th_.size() + 1; }
  template <class F>
  void run(int n, F&& f) {
    if (n <= 1 || th_.empty()) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    // `left` lives on this frame: a task's decrement is its last access to
    // it, so the caller may return as soon as it reads zero
    std::atomic<int> left{n};
    auto one = [&](int i) {
      f(i);
      left.fetch_sub(1, std::memory_order_acq_rel);
    };
    {
      std::lock_guard<std::mutex> g(mu_);
      for (int i = 1; i < n; ++i) q_.push_back([&one, i] { one(i); });
      pending_.fetch_add(n - 1, std::memory_order_release);
    }
    if (sleepers_.load(std::memory_order_acquire) > 0) cv_.notify_all();
    one(0);
    std::function<void()> t;
    while (pop(t)) t();  // help: ours or another caller's tasks
    for (int k = 0; left.load(std::memory_order_acquire) != 0; ++k) pause(k);
  }

 private:
  static void pause(int k) {
#if defined(__x86_64__)
    if (k < 4096) {
      _mm_pause();
      return;
    }
#endif
    std::this_thread::yield();
  }
  bool pop(std::function<void()>& t) {
    if (pending_.load(std::memory_order_acquire) == 0) return false;
    std::lock_guard<std::mutex> g(mu_);
    if (q_.empty()) return false;
    t = std::move(q_.front());
    q_.pop_front();
    pending_.fetch_sub(1, std::memory_order_relaxed);
    return true;
  }
  void worker() {
    using clk = std::chrono::steady_clock;
    for (;;) {
      std::function<void()> t;
      if (pop(t)) {
        t();
        continue;
      }
      // spin ~0.5 ms for the next chunk before sleeping
      const auto t0 = clk::now();
      bool more = false;
      for (int k = 0;; ++k) {
        if (pending_.load(std::memory_order_acquire) > 0) {
          more = true;
          break;
        }
#if defined(__x86_64__)
        _mm_pause();
#endif
        if ((k & 255) == 255 && clk::now() - t0 > std::chrono::microseconds(500)) break;
      }
      if (more) continue;
      std::unique_lock<std::mutex> g(mu_);
      sleepers_.fetch_add(1, std::memory_order_acq_rel);
      cv_.wait(g, [&] { return !q_.empty(); });
      sleepers_.fetch_sub(1, std::memory_order_acq_rel);
      t = std::move(q_.front());
      q_.pop_front();
      pending_.fetch_sub(1, std::memory_order_relaxed);
      g.unlock();
      t();
    }
  }
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    int n = (int)std::min(hw, 16u) - 1;
    if (const char* e = std::getenv("VK_RL_HOST_THREADS")) n = std::max(0, std::atoi(e) - 1);
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { worker(); });
    for (auto& t : th_) t.detach();
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  std::atomic<int> pending_{0}, sleepers_{0};
  std::vector<std::thread> th_;
};

// memcpy with non-temporal (streaming) stores.  A staging chunk written by
// ordinary stores from many pool threads is left as dirty lines in those
// cores' private caches; once the threads go idle, the DMA that reads the
// chunk has to snoop them out of sleeping cores, and the last chunk of a call
// measured 1.9-2.8 ms instead of 0.32 ms for 16 MB (profiles/r02/staging_dma.md).
// Streaming stores put the bytes in DRAM instead.
void copy_nt(void* dst, const void* src, size_t n) {
#if defined(__x86_64__)
  char* d = (char*)dst;
  const char* s = (const char*)src;
  size_t head = (16 - ((uintptr_t)d & 15)) & 15;
  if (head > n) head = n;
  std::memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  const size_t nv = n / 64;
  for (size_t i = 0; i < nv; ++i, s += 64, d += 64) {
    const __m128i a = _mm_loadu_si128((const __m128i*)s), b = _mm_loadu_si128((const __m128i*)(s + 16));
    const __m128i c = _mm_loadu_si128((const __m128i*)(s + 32)), e = _mm_loadu_si128((const __m128i*)(s + 48));
    _mm_stream_si128((__m128i*)d, a);
    _mm_stream_si128((__m128i*)(d + 16), b);
    _mm_stream_si128((__m128i*)(d + 32), c);
    _mm_stream_si128((__m128i*)(d + 48), e);
  }
  std::memcpy(d, s, n - nv * 64);
  _mm_sfence();
#else
  std::memcpy(dst, src, n);
#endif
}

bool nt_copy_on() {
  static const bool on = [] {
    const char* e = std::getenv("VK_RL_NT_COPY");
    return !(e && e[0] == '0');
  }();
  return on;
}

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = 1 << 20;
  HostPool& pool = HostPool::get();
  const bool nt = nt_copy_on();
  auto cp = [nt](void* d, const void* s, size_t n) {
    if (nt)
      copy_nt(d, s, n);
    else
      std::memcpy(d, s, n);
  };
  const int n = (int)std::min<size_t>((size_t)pool.size(), (bytes + kPiece - 1) / kPiece);
  if (n <= 1) {
    cp(dst, src, bytes);
    return;
  }
  const size_t per = (bytes / n + 63) / 64 * 64;
  pool.run(n, [&](int i) {
    const size_t off = (size_t)i * per;
    if (off < bytes) cp((char*)dst + off, (const char*)src + off, std::min(per, bytes - off));
  });
}

// Faults in the pages of a fresh pageable output buffer (one write per page,
// split over the pool), so the copy-out after the run does not page-fault.
void prefault(void* dst, size_t bytes) {
  constexpr size_t kPage = 4096, kPiece = 8 << 20;
  HostPool& pool = HostPool::get();
  const int n = (int)std::max<size_t>(1, std::min<size_t>((size_t)pool.size(), bytes / kPiece));
  const size_t per = (bytes / n + kPage - 1) / kPage * kPage;
  pool.run(n, [&](int i) {
    volatile char* b = (volatile char*)dst;
    for (size_t o = (size_t)i * per; o < std::min(bytes, (size_t)(i + 1) * per); o += kPage) b[o] = 0;
  });
}

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

struct Staging {
  static constexpr int kMaxSlots = 16;
  // ring geometry: VK_RL_STAGE_MB (chunk size) x VK_RL_STAGE_SLOTS
  const int kSlots = [] {
    const char* e = std::getenv("VK_RL_STAGE_SLOTS");
    return e ? std::max(2, std::min(kMaxSlots, std::atoi(e))) : 4;
  }();
  const size_t kChunk = [] {
    const char* e = std::getenv("VK_RL_STAGE_MB");
    return (size_t)(e ? std::max(1, std::atoi(e)) : 16) << 20;
  }();
  void* h[kMaxSlots]{};
  cudaEvent_t ev[kMaxSlots]{};
  ~Staging() {
    for (int i = 0; i < kSlots; ++i) {
      if (h[i]) cudaFreeHost(h[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
  }
  void ensure() {
    for (int i = 0; i < kSlots; ++i) {
      if (!h[i]) ck(cudaMallocHost(&h[i], kChunk), "pinned staging");
      if (!ev[i]) ck(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "staging event");
    }
  }
  // host -> device, enqueued on s; returns when every host byte has been read
  void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (host_pinned(src)) {
      ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "H2D");
      return;
    }
    ensure();
    const bool tm = timing_on();
    std::vector<cudaEvent_t> te;  // VK_RL_TIMING: per-chunk DMA times
    std::vector<double> cpy;
    const size_t cs = kChunk;
    size_t off = 0;
    for (int c = 0; off < bytes; ++c, off += cs) {
      const int k = c % kSlots;
      const size_t n = std::min(cs, bytes - off);
      if (c >= kSlots) ck(cudaEventSynchronize(ev[k]), "staging");  // slot's previous DMA done
      const auto t0 = std::chrono::steady_clock::now();
      parallel_memcpy(h[k], (const char*)src + off, n);
      if (tm) {
        cpy.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        te.resize(te.size() + 2);
        cudaEventCreate(&te[te.size() - 2]);
        cudaEventCreate(&te[te.size() - 1]);
        cudaEventRecord(te[te.size() - 2], s);
      }
      ck(cudaMemcpyAsync((char*)dst + off, h[k], n, cudaMemcpyHostToDevice, s), "H2D");
      if (tm) cudaEventRecord(te.back(), s);
      ck(cudaEventRecord(ev[k], s), "staging");
    }
    if (tm) {
      cudaStreamSynchronize(s);
      std::fprintf(stderr, "  h2d chunks (host copy / DMA ms):");
      for (size_t i = 0; i < cpy.size(); ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, te[2 * i], te[2 * i + 1]);
        std::fprintf(stderr, " %.3f/%.3f", cpy[i], ms);
        cudaEventDestroy(te[2 * i]);
        cudaEventDestroy(te[2 * i + 1]);
      }
      std::fprintf(stderr, "\n");
    }
  }
  // device -> host after everything enqueued on s; returns when dst is written
  void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (host_pinned(dst)) {
      ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaStreamSynchronize(s), "D2H");
      return;
    }
    ensure();
    const size_t cs = kChunk;
    const int nc = (int)((bytes + cs - 1) / cs);
    auto issue = [&](int c) {
      const int k = c % kSlots;
      const size_t off = (size_t)c * cs, n = std::min(cs, bytes - off);
      ck(cudaMemcpyAsync(h[k], (const char*)src + off, n, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaEventRecord(ev[k], s), "staging");
    };
    for (int c = 0; c < std::min(nc, kSlots); ++c) issue(c);
    for (int c = 0; c < nc; ++c) {
      const int k = c % kSlots;
      const size_t off = (size_t)c * cs, n = std::min(cs, bytes - off);
      ck(cudaEventSynchronize(ev[k]), "D2H");
      parallel_memcpy((char*)dst + off, h[k], n);
      if (c + kSlots < nc) issue(c + kSlots);
    }
  }
};

constexpr size_t kSmemCap = 110 * 1024;  // two CTAs per SM
constexpr int kThreads = 256;
constexpr int kFrcBlocks = 148 * 6;  // FRC ring-sum blocks (per-block partials, fixed-order reduce)

}  // namespace

struct vk_rl_plan_s {
  int device = 0;
  int rank = 3;
  bool pad = true;
  int conv = 0;  // 0: RL plan; 1 / 2: filters::fft_convolve plan, linear / circular
  // circular fft_convolve on extents that are not 5-smooth: a linear plan on
  // the periodic extension E = A + K - 1 (offset h = K-1-c), see conv_device
  vk_rl_plan_s* circ = nullptr;
  int circ_h[3]{}, circ_e[3]{};
  DevBuf<float> circ_in, circ_out;
  // slab plans (vk_rl_slab_*): own P rows [own0, own1) of the local domain;
  // halo rows below / above are refreshed by the caller between passes
  bool slab = false;
  int own0 = 0, own1 = 0;
  uint64_t ishape[3]{}, dshape[3]{}, wshape[3]{}, kshape[3]{};
  Geom g{};
  int Kz = 1, Ky = 1, Kx = 1;
  int psf_status = 0;  // 0 ok, VK_ERR_NEGATIVE, VK_ERR_UNNORMALIZED_PSF
  std::string psf_msg;

  DevBuf<float2> twx, twy, twz, twx2, twy2, twz2;
  LinePlan lpx{}, lpy{}, lpz{};
  // compile-time-length kernels per axis (nullptr -> generic Stockham)
  const vk::FastEntry* fx = nullptr;
  const vk::FastEntry* fy = nullptr;
  const vk::FastEntry* fz = nullptr;
  // TMA descriptor of S_B for the z convolution (zpass_tma), when available
  bool ztma = false, otma = false, ytma = false;
  int xpf = 0;  // x-pass L2 prefetch mask (XArgs::pf)
  int ycrop = 0;
  bool xtma = false;  // xpass_tma for the RATIO/UPDATE x passes (S_A rows staged by TMA)
  CUtensorMap xmap{};
  int xtbk = 0, xtnb = 0;  // crop offset of the y inverse: g.cy, or 0 when folded into the OTFs as a ramp
  bool tma_store = true;  // TMA/bulk stores of the z tile and y-forward lines (VK_RL_NO_TMA_STORE=1: thread stores)  // S_A kx-blocked by 1 << blk_lb (= the y pass's lines per CTA); 0: [Hx][Pz][Py]
  CUtensorMap zmap{}, omap{}, omap_flip{};
  // kx-chunked y/z convolution (conv_yz_chunked): chunks of kxc planes run
  // y-forward -> z -> y-inverse through a ring slot (one per stream) small
  // enough to stay L2-resident, so S_B does not make HBM round trips
  int kxc = 0, kxs = 3;  // planes per chunk, streams (= ring slots)
  int kxn = 0;           // chunks; boundaries kx0 = c * Hx / kxn (sizes differ by <= 1)
  size_t ring_window = 0;  // bytes of ring2 under a persisting L2 access window (0: none)
  DevBuf<float2> ring2;
  CUtensorMap zmap_ring[4]{};
  cudaStream_t kstream[4]{};  // kstream[0] unused (the run's stream)
  // device-side stopping: the iteration body as a CUDA graph under a WHILE
  // conditional node whose condition the rule kernel sets (run_graph_loop)
  cudaGraph_t gr = nullptr;
  cudaGraphExec_t grx = nullptr;
  struct GraphKey {
    const float* obs = nullptr;
    int metric = -1, iters = 0, patience = 0;
    double rel_tol = 0, spacing = 0;
    bool operator==(const GraphKey& o) const {
      return obs == o.obs && metric == o.metric && iters == o.iters && patience == o.patience &&
             (rel_tol == o.rel_tol || (rel_tol != rel_tol && o.rel_tol != o.rel_tol)) && spacing == o.spacing;
    }
  } grkey;
  uint64_t gr_body_launches = 0;
  DevBuf<vk::StopState> gstate;
  DevBuf<double> gvalues, gmetric;
  DevBuf<unsigned long long> gts;
  DevBuf<unsigned> grange_init;
  cudaEvent_t kev[4]{};
  // frc_resolution stopping metric (rl_metrics.cuh): a sub-plan supplies the
  // r2c transforms of the two half-size checkerboard images
  vk_rl_plan_s* frc = nullptr;
  DevBuf<float> frc_even, frc_odd;
  DevBuf<double> frc_bins;
  double* h_frc = nullptr;  // pinned [3][nbins]
  int frc_nbins = 0, frc_slices = 1;
  double frc_binf = 0;
  int frc_h[3]{1, 1, 1}, frc_s[3]{0, 0, 0};
  // non-5-smooth half extents: direct per-axis DFTs instead of the sub-plan
  bool frc_dft = false;
  DevBuf<float2> frc_tw[3], frc_t1, frc_A, frc_B;
  // ssim_vs_prev stopping metric (rl_metrics.cuh): current / previous crops
  // (ping-pong), two sets of five double moment fields, per-iteration crop
  // ranges ([iters+1][2] f32 bits, row 0 = observed) and SSIM-map sums
  DevBuf<float> ss_img[2];
  DevBuf<double> ss_f[2];
  DevBuf<unsigned> ss_range;
  DevBuf<double> ss_sum;
  int ss_cap = 0;
  bool ss_ready = false;
  int xL = 1, yL = 1, zL = 1;
  size_t xs = 0, ys = 0, zs = 0;

  DevBuf<float2> SA, SB, otf, otf_flip;
  DevBuf<float2> ofac;  // 1D factors of otf and otf_flip when both are separable (ZTmaArgs::ofac)
  bool ofactored = false;
  // ky-mirror-symmetric OTFs (halve_otfs): only columns ky <= Wy/2 stored,
  // [Hx][Wz][owp] with owp = Wy/2+1 rounded up to even (16-byte TMA pitch)
  bool ohalf = false;
  int owp = 0;
  DevBuf<float> est, obs, out;
  DevBuf<double> acc;
  DevBuf<vk::ObsStats> stats;
  int acc_cap = 0;
  // deterministic sums (rl_passes.cuh block_partial): x-pass block partials
  // of the last kSumRing iterations [slot][xblocks][4], reduced into acc in a
  // fixed order by flush_sums(); sum_done = iterations already in acc
  DevBuf<double> xpart, part;
  int xblocks = 0, sum_done = 0;

  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> events;
  double* h_acc = nullptr;  // pinned
  uint64_t launches = 0;
  Staging staging;  // pinned chunks for pageable host buffers
  bool cached = false, busy = false;  // plan cache (vk_richardson_lucy & co.)

  // Optional per-launch CUDA-event timing, by kernel kind (vk_rl_plan_profile).
  bool prof = false;
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
  struct ProfRec {
    int kind;
    size_t ev;           // index of the begin event
    double bytes, otf;   // algorithmic and OTF bytes of this launch
  };
  std::vector<ProfRec> prof_pending;
  double prof_ms[VK_KIND_COUNT]{};
  uint64_t prof_n[VK_KIND_COUNT]{};
  double prof_bytes[VK_KIND_COUNT]{}, prof_otf[VK_KIND_COUNT]{};
  double prof_last_otf[VK_KIND_COUNT]{};  // OTF bytes per launch of the last profile read (-1: none)

  // Batch lanes: clones of this plan (own buffers and stream) that run
  // independent volumes concurrently, one host thread each (lane 0 = this).
  std::vector<float> psf_host;
  std::vector<vk_rl_plan_s*> lanes;

  ~vk_rl_plan_s() {
    for (auto* l : lanes) delete l;
    for (auto e : events) cudaEventDestroy(e);
    for (auto e : prof_pool) cudaEventDestroy(e);
    if (h_acc) cudaFreeHost(h_acc);
    if (stream) cudaStreamDestroy(stream);
    if (h_frc) cudaFreeHost(h_frc);
    if (grx) cudaGraphExecDestroy(grx);
    if (gr) cudaGraphDestroy(gr);
    for (int i = 0; i < 4; ++i) {
      if (kstream[i]) cudaStreamDestroy(kstream[i]);
      if (kev[i]) cudaEventDestroy(kev[i]);
    }
    delete frc;
    delete circ;
  }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void launch_check(vk_rl_plan p, const char* what) {
  ++p->launches;
  ck(cudaGetLastError(), what);
}

// Per-launch event bracketing when profiling is on (records on the launch
// stream, so it sees exactly the kernel's device time).
size_t prof_begin(vk_rl_plan p, cudaStream_t s) {
  if (!p->prof) return 0;
  while (p->prof_pool.size() < p->prof_used + 2) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event");
    p->prof_pool.push_back(e);
  }
  const size_t i = p->prof_used;
  p->prof_used += 2;
  ck(cudaEventRecord(p->prof_pool[i], s), "event");
  return i;
}
uint64_t alg_bytes(vk_rl_plan p, int kind);
uint64_t otf_bytes(vk_rl_plan p, int kind);

// bytes < 0: the kind's whole-volume launch (alg_bytes / otf_bytes); chunked
// launches pass their own (otf as the fraction of the OTF planes they read).
void prof_end(vk_rl_plan p, cudaStream_t s, int kind, size_t i, double bytes = -1.0, double otf_frac = 1.0) {
  if (!p->prof) return;
  ck(cudaEventRecord(p->prof_pool[i + 1], s), "event");
  p->prof_pending.push_back({kind, i, bytes < 0 ? (double)alg_bytes(p, kind) : bytes,
                             otf_frac * (double)otf_bytes(p, kind)});
}
void prof_collect(vk_rl_plan p) {
  for (const auto& r : p->prof_pending) {
    const int kind = r.kind;
    const size_t i = r.ev;
    ck(cudaEventSynchronize(p->prof_pool[i + 1]), "event sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, p->prof_pool[i], p->prof_pool[i + 1]), "elapsed");
    p->prof_ms[kind] += ms;
    p->prof_n[kind] += 1;
    p->prof_bytes[kind] += r.bytes;
    p->prof_otf[kind] += r.otf;
  }
  p->prof_pending.clear();
  p->prof_used = 0;
}

constexpr int kSumRing = 16;   // iterations of x-pass partials kept before a reduce
constexpr int kStatBlocks = 148 * 4;  // grid of the grid-stride statistics kernels

// Reduces the x-pass partials of iterations sum_done+1 .. upto (1-based) into
// acc[it-1][0..3], in a fixed order.
void flush_sums(vk_rl_plan p, cudaStream_t s, int upto) {
  if (upto <= p->sum_done) return;
  const int n = upto - p->sum_done;
  vk::reduce_iter_partials_kernel<<<4 * n, 256, 0, s>>>(p->xpart.p, p->xblocks, kSumRing, p->sum_done, p->acc.p);
  launch_check(p, "reduce sums");
  p->sum_done = upto;
}

// ---- pass launchers -------------------------------------------------------

// pdl: programmatic dependent launch (the kernel calls pdl_trigger/pdl_wait,
// rl_fast.cuh); VK_RL_NO_PDL=1 turns it off.
thread_local bool t_capturing = false;  // inside run_graph_loop's stream capture

void launch(const void* k, dim3 grid, int nt, size_t smem, cudaStream_t s, void* arg, bool pdl = false) {
  void* args[] = {arg};
  static const bool no_pdl = [] {
    const char* e = std::getenv("VK_RL_NO_PDL");
    return e && e[0] == '1';
  }();
  if (!pdl || no_pdl || t_capturing) {  // graph body: plain kernel nodes
    ck(cudaLaunchKernel(k, grid, dim3(nt), args, smem, s), "launch");
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ck(cudaLaunchKernelExC(&cfg, k, args), "launch");
}

// zoff / nz: z rows [zoff, zoff + nz) only (z-chunked iterations; nz < 0 = all)
// it: the RL iteration (1-based) whose sums this RATIO / UPDATE pass produces
// (block partials into ring slot (it-1) % kSumRing); 0 for the other modes.
void x_pass(vk_rl_plan p, cudaStream_t s, int mode, const float* src, int rows_z, int rows_y, int len,
            float scale, float* est, const float* obs, int it, float* out, int xoff = 0, int zoff = 0,
            int nz = -1) {
  vk::XArgs a{};
  a.zoff = zoff;
  a.plan = p->lpx;
  a.g = p->g;
  a.mode = mode;
  a.L = p->fx ? p->fx->Lx : p->xL;
  a.xoff = xoff;
  a.rows_z = rows_z;
  a.rows_y = rows_y;
  a.len = len;
  a.S = p->SA.p;
  a.src = src;
  a.scale = scale;
  a.est = est;
  a.obs = obs;
  a.acc = nullptr;
  if (it > 0) {
    // the slot of iteration it last held iteration it - kSumRing: reduce first
    if (it - kSumRing > p->sum_done) flush_sums(p, s, it - 1);
    a.acc = p->xpart.p + (size_t)((it - 1) % kSumRing) * p->xblocks * 4;
  }
  a.out = out;
  a.pf = p->xpf;
  dim3 grid((rows_y + 2 * a.L - 1) / (2 * a.L), nz < 0 ? rows_z : nz);
  const int kind = mode == vk::XM_FWD ? VK_KIND_X_FWD : mode == vk::XM_RATIO ? VK_KIND_X_RATIO : VK_KIND_X_UPDATE;
  const size_t t = prof_begin(p, s);
  if (p->fx && p->xtma && mode != vk::XM_FWD) {
    vk::XTmaArgs ta{};
    ta.map = p->xmap;
    a.tbk = p->xtbk;
    a.tnb = p->xtnb;
    ta.x = a;
    launch(p->fx->xtk, grid, p->fx->NTx, p->fx->smem_xp, s, &ta, p->fx->pdl);
  } else if (p->fx)
    launch(p->fx->xk, grid, p->fx->NTx, p->fx->smem_xp, s, &a, p->fx->pdl);
  else
    vk::xpass_kernel<<<grid, kThreads, p->xs, s>>>(a);
  launch_check(p, "xpass");
  prof_end(p, s, kind, t);
}

// zcn > 0: only the lines (kx, z) with z in [zc0, zc0 + zcn) of zrows per kx
// plane (nlines is then Hx * zcn)
void y_pass(vk_rl_plan p, cudaStream_t s, int mode, int nlines, int n_in, int in_pitch, int n_out,
            int out_pitch, int out_off, const float2* in, float2* out, const float2* otf, int zc0 = 0, int zcn = 0,
            int zrows = 0) {
  vk::YArgs a{};
  a.zc0 = zc0;
  a.zcn = zcn;
  a.zrows = zrows;
  a.plan = p->lpy;
  a.mode = mode;
  a.L = p->fy ? p->fy->Ly : p->yL;
  a.nlines = nlines;
  a.n_in = n_in;
  a.in_pitch = in_pitch;
  a.n_out = n_out;
  a.out_pitch = out_pitch;
  a.out_off = out_off;
  a.in = in;
  a.out = out;
  a.otf = otf;
  dim3 grid((nlines + a.L - 1) / a.L);
  const int kind = mode == vk::YM_FWD ? VK_KIND_Y_FWD : mode == vk::YM_INV ? VK_KIND_Y_INV : VK_KIND_Y_CONV;
  const size_t t = prof_begin(p, s);
  if (p->fy)
  {
    a.bst = p->tma_store && out_off % 2 == 0 && out_pitch % 2 == 0 && n_out % 2 == 0 &&
            (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    if (p->ytma && n_in % 2 == 0 && in_pitch % 2 == 0) {
      if (mode == vk::YM_CONV && p->ofactored && p->g.Wz == 1 && a.zcn == 0) {
        const size_t nf = (size_t)p->g.Hx + p->g.Wy + p->g.Wz;
        a.ofac = otf == p->otf.p ? p->ofac.p : otf == p->otf_flip.p ? p->ofac.p + nf : nullptr;
        a.ohx = p->g.Hx;
      }
      launch(p->fy->ytk, grid, p->fy->NTy, p->fy->smem_yt, s, &a, p->fy->pdl);
    }
    else
      launch(p->fy->yk, grid, p->fy->NTy, mode == vk::YM_CONV ? p->fy->smem_yconv : p->fy->smem_yp, s, &a,
             p->fy->pdl);
  }
  else
    vk::ypass_kernel<<<grid, kThreads, p->ys, s>>>(a);
  launch_check(p, "ypass");
  prof_end(p, s, kind, t, 8.0 * nlines * (n_in + n_out));
}

void z_pass(vk_rl_plan p, cudaStream_t s, int mode, int zrows, int n_in, int n_out, int out_off,
            float2* S, const float2* otf, float2* otf_out) {
  vk::ZArgs a{};
  a.plan = p->lpz;
  a.mode = mode;
  a.L = p->fz ? p->fz->Lz : p->zL;
  a.Wy = p->g.Wy;
  a.zrows = zrows;
  a.n_in = n_in;
  a.n_out = n_out;
  a.out_off = out_off;
  a.S = S;
  a.otf = otf;
  a.otf_out = otf_out;
  a.hx = p->g.Hx;
  if (p->fz && p->ztma && mode == vk::ZM_CONV && S == p->SB.p && zrows == p->g.Pz && n_in == p->g.Pz) {
    vk::ZTmaArgs ta{};
    ta.map = p->zmap;
    ta.z = a;
    ta.otf_tma = p->otma && (otf == p->otf.p || otf == p->otf_flip.p);
    ta.tma_store = p->tma_store && n_out == p->g.Pz;
    if (p->ofactored) {
      const size_t nf = (size_t)p->g.Hx + p->g.Wy + p->g.Wz;
      ta.ofac = otf == p->otf.p ? p->ofac.p : otf == p->otf_flip.p ? p->ofac.p + nf : nullptr;
      if (ta.ofac) ta.otf_tma = 0;
    }
    if (ta.otf_tma) ta.omap = otf == p->otf.p ? p->omap : p->omap_flip;
    ta.otf_half = ta.otf_tma && p->ohalf;
    dim3 grid((p->g.Wy + 15) / 16, p->g.Hx);
    const size_t t = prof_begin(p, s);
    launch(p->fz->ztk, grid, p->fz->NTz, ta.otf_half ? p->fz->smem_zt_half : p->fz->smem_zt, s, &ta, p->fz->pdl);
    launch_check(p, "zpass tma");
    prof_end(p, s, VK_KIND_Z_CONV, t);
    return;
  }
  dim3 grid((p->g.Wy + a.L - 1) / a.L, p->g.Hx);
  const size_t t = prof_begin(p, s);
  if (p->fz)
    launch(p->fz->zk, grid, p->fz->NTz, p->fz->smem_z, s, &a, p->fz->pdl);
  else
    vk::zpass_kernel<<<grid, kThreads, p->zs, s>>>(a);
  launch_check(p, "zpass");
  prof_end(p, s, VK_KIND_Z_CONV, t);
}

// z convolution of kx planes [kx0, kx0 + nk) held in ring slot `slot`.
void z_pass_chunk(vk_rl_plan p, cudaStream_t s, const float2* otf, int kx0, int nk, int slot) {
  vk::ZTmaArgs ta{};
  ta.map = p->zmap_ring[slot];
  ta.z.plan = p->lpz;
  ta.z.mode = vk::ZM_CONV;
  ta.z.L = 16;
  ta.z.Wy = p->g.Wy;
  ta.z.zrows = p->g.Pz;
  ta.z.n_in = p->g.Pz;
  ta.z.n_out = p->g.Pz;
  ta.z.out_off = p->g.cz;
  ta.z.S = p->ring2.p + (size_t)slot * p->kxc * p->g.Pz * p->g.Wy;
  ta.z.otf = otf;
  ta.z.hx = p->g.Hx;
  ta.kx0 = kx0;
  ta.otf_tma = p->otma && (otf == p->otf.p || otf == p->otf_flip.p);
  ta.tma_store = 1;
  if (p->ofactored) {
    const size_t nf = (size_t)p->g.Hx + p->g.Wy + p->g.Wz;
    ta.ofac = otf == p->otf.p ? p->ofac.p : otf == p->otf_flip.p ? p->ofac.p + nf : nullptr;
    if (ta.ofac) ta.otf_tma = 0;
  }
  if (ta.otf_tma) ta.omap = otf == p->otf.p ? p->omap : p->omap_flip;
  ta.otf_half = ta.otf_tma && p->ohalf;
  const size_t t = prof_begin(p, s);
  launch(p->fz->ztk, dim3((p->g.Wy + 15) / 16, nk), p->fz->NTz, ta.otf_half ? p->fz->smem_zt_half : p->fz->smem_zt, s,
         &ta, p->fz->pdl);
  launch_check(p, "zpass chunk");
  prof_end(p, s, VK_KIND_Z_CONV, t, 16.0 * nk * p->g.Pz * p->g.Wy, (double)nk / p->g.Hx);
}

// The y/z convolution in chunks of kxc kx planes: y-forward -> z -> y-inverse
// per chunk through an L2-sized ring slot, chunk c on stream c % kxs (the
// run's stream and kxs-1 forked ones, joined at the end), so the chunks'
// passes overlap and fill the GPU while each chunk's S_B stays in L2
// (C2: 11 chunks of 27 planes, 21 MB each, instead of 210 MB of S_B making
// two HBM round trips per convolution; profiles/r02/kxchunk.md).
void conv_yz_chunked(vk_rl_plan p, cudaStream_t s, const float2* otf) {
  const Geom& g = p->g;
  const int ns = p->kxs;
  if (!p->kev[0]) {
    for (int i = 0; i < p->kxs; ++i) {
      if (i) ck(cudaStreamCreateWithFlags(&p->kstream[i], cudaStreamNonBlocking), "cudaStreamCreate");
      ck(cudaEventCreateWithFlags(&p->kev[i], cudaEventDisableTiming), "event");
    }
    if (p->ring_window) {  // keep the ring L2-resident (persisting access window)
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = p->ring2.p;
      v.accessPolicyWindow.num_bytes = p->ring_window;
      v.accessPolicyWindow.hitRatio = 1.0f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      for (int i = 1; i < p->kxs; ++i) cudaStreamSetAttribute(p->kstream[i], cudaStreamAttributeAccessPolicyWindow, &v);
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
      cudaGetLastError();
    }
  }
  ck(cudaEventRecord(p->kev[0], s), "event");
  for (int i = 1; i < ns; ++i) ck(cudaStreamWaitEvent(p->kstream[i], p->kev[0], 0), "wait");
  const size_t plane_a = (size_t)g.Pz * g.Py, slot_b = (size_t)p->kxc * g.Pz * g.Wy;
  int c = 0;
  for (int kx0 = 0; kx0 < g.Hx; ++c) {
    const int kx1 = p->kxn ? (int)((long long)(c + 1) * g.Hx / p->kxn) : std::min(kx0 + p->kxc, g.Hx);
    const int nk = kx1 - kx0, slot = c % ns;
    cudaStream_t cs = slot ? p->kstream[slot] : s;
    float2* sa = p->SA.p + (size_t)kx0 * plane_a;
    float2* sb = p->ring2.p + (size_t)slot * slot_b;
    y_pass(p, cs, vk::YM_FWD, nk * g.Pz, g.Py, g.Py, g.Wy, g.Wy, 0, sa, sb, nullptr);
    z_pass_chunk(p, cs, otf, kx0, nk, slot);
    y_pass(p, cs, vk::YM_INV, nk * g.Pz, g.Wy, g.Wy, g.Py, g.Py, p->ycrop, sb, sa, nullptr);
    kx0 = kx1;
  }
  for (int i = 1; i < ns; ++i) {
    ck(cudaEventRecord(p->kev[i], p->kstream[i]), "event");
    ck(cudaStreamWaitEvent(s, p->kev[i], 0), "wait");
  }
}

// 'same' linear convolution of the x-transformed P-domain field held in SA
// with `otf` (deconv.cpp:135-147 minus the x transforms, which live in the
// fused X-pass).  Result back in SA.
void conv_yz(vk_rl_plan p, cudaStream_t s, const float2* otf) {
  const Geom& g = p->g;
  const int nl = g.Hx * g.Pz;
  if (g.Wz == 1) {
    y_pass(p, s, vk::YM_CONV, nl, g.Py, g.Py, g.Py, g.Py, p->ycrop, p->SA.p, p->SA.p, otf);
    return;
  }
  // profiled runs take the whole-volume passes: chunk launches on several
  // streams overlap, so per-launch events could not attribute time to kernels
  if (p->kxc && !p->prof) {
    conv_yz_chunked(p, s, otf);
    return;
  }
  y_pass(p, s, vk::YM_FWD, nl, g.Py, g.Py, g.Wy, g.Wy, 0, p->SA.p, p->SB.p, nullptr);
  z_pass(p, s, vk::ZM_CONV, g.Pz, g.Pz, g.Pz, g.cz, p->SB.p, otf, nullptr);
  y_pass(p, s, vk::YM_INV, nl, g.Wy, g.Wy, g.Py, g.Py, p->ycrop, p->SB.p, p->SA.p, nullptr);
}

// Full r2c spectrum [Hx][Wz][Wy] of a real block [rz][ry][rx] corner-embedded
// in the plan's W grid, times `scale`.
void spectrum3d(vk_rl_plan p, cudaStream_t s, const float* d_src, int rz, int ry, int rx, float scale,
                float2* dst) {
  const Geom& g = p->g;
  x_pass(p, s, vk::XM_FWD, d_src, rz, ry, rx, scale, nullptr, nullptr, 0, nullptr);
  const int nl = g.Hx * rz;
  if (g.Wz == 1) {
    y_pass(p, s, vk::YM_FWD, nl, ry, ry, g.Wy, g.Wy, 0, p->SA.p, dst, nullptr);
    return;
  }
  y_pass(p, s, vk::YM_FWD, nl, ry, ry, g.Wy, g.Wy, 0, p->SA.p, p->SB.p, nullptr);
  z_pass(p, s, vk::ZM_FWD_OUT, rz, rz, 0, 0, p->SB.p, nullptr, dst);
}

// OTF of a corner-embedded PSF on the W grid, 1/prod(W) folded in
// (deconv.cpp:126-130 + fft_plan.cpp:95-96).
void build_otf(vk_rl_plan p, const float* d_psf, float2* otf_dst) {
  const Geom& g = p->g;
  const float scale = (float)(1.0 / ((double)g.Wz * g.Wy * g.Wx));
  spectrum3d(p, p->stream, d_psf, p->Kz, p->Ky, p->Kx, scale, otf_dst);
}

// ---- factored OTF (separable PSF) ----------------------------------------
// A separable PSF has a separable OTF; the per-axis crop ramps are separable
// too.  Then O(kx, kz, ky) = O(kx,0,0) O(0,kz,0) O(0,0,ky) / O(0,0,0)^2, and
// the TMA z pass rebuilds each OTF column from three 1D factors instead of
// reading the OTF (C4: 673 MB per z launch).  The rank-1 property is TESTED
// on the device OTF, not assumed from the PSF: max |O - product| must be
// <= kOtfSepTol * max |O| for both OTFs.
constexpr float kOtfSepTol = 4e-6f;

__global__ void otf_factor_kernel(const float2* __restrict__ otf, int Hx, int Wz, int Wy, float2* __restrict__ fac) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t plane = (size_t)Wz * Wy;
  if (i < Hx) {  // fx = O(kx,0,0) / O000^2, in double
    const double2 o = make_double2(otf[0].x, otf[0].y);
    const double2 o2 = make_double2(o.x * o.x - o.y * o.y, 2.0 * o.x * o.y);
    const double d = o2.x * o2.x + o2.y * o2.y;
    const float2 v = otf[(size_t)i * plane];
    fac[i] = d > 0.0 ? make_float2((float)((v.x * o2.x + v.y * o2.y) / d), (float)((v.y * o2.x - v.x * o2.y) / d))
                     : make_float2(0.f, 0.f);
  } else if (i < Hx + Wy) {
    fac[i] = otf[i - Hx];  // fy = O(0,0,ky)
  } else if (i < Hx + Wy + Wz) {
    fac[i] = otf[(size_t)(i - Hx - Wy) * Wy];  // fz = O(0,kz,0)
  }
}

// bits[0] = max |O - (fx fy) fz|, bits[1] = max |O| (non-negative floats as uint)
__global__ void otf_sep_check_kernel(const float2* __restrict__ otf, const float2* __restrict__ fac, int Hx, int Wz,
                                     int Wy, unsigned* bits) {
  const size_t n = (size_t)Hx * Wz * Wy;
  const float2* fy = fac + Hx;
  const float2* fz = fac + Hx + Wy;
  float err = 0.f, mx = 0.f;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int ky = (int)(i % Wy);
    const size_t r = i / Wy;
    const int kz = (int)(r % Wz), kx = (int)(r / Wz);
    const float2 o = otf[i];
    const float2 q = vk::cmul(vk::cmul(fac[kx], fy[ky]), fz[kz]);
    err = fmaxf(err, hypotf(o.x - q.x, o.y - q.y));
    mx = fmaxf(mx, hypotf(o.x, o.y));
  }
  for (int m = 16; m > 0; m >>= 1) {
    err = fmaxf(err, __shfl_xor_sync(0xffffffffu, err, m));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&bits[0], __float_as_uint(err));
    atomicMax(&bits[1], __float_as_uint(mx));
  }
}

// ---- half OTF (ky-mirror-symmetric PSF) ----------------------------------------
// With both crop ramps folded in, the OTF of a PSF that is mirror-symmetric
// along y (odd Ky) is EVEN in ky: the y ramp e^{+2 pi i cy ky / Wy} cancels
// the corner-embedding phase e^{-2 pi i ky (Ky-1)/2 / Wy} exactly and what is
// left is the transform of a centred symmetric function.  The widefield PSF
// of C2 (and any PSF symmetric in y) qualifies -- it is not separable, so
// the z pass reads its OTF -- and then only the Wy/2+1 columns ky <= Wy/2 are
// stored and read: 128 of 256 MB per C2 z launch.  TESTED on the device OTFs
// like the factored form: max |O(ky) - O(Wy-ky)| <= kOtfSepTol * max |O|.
__global__ void otf_mirror_check_kernel(const float2* __restrict__ otf, int Hx, int Wz, int Wy, unsigned* bits) {
  const size_t n = (size_t)Hx * Wz * Wy;
  float err = 0.f, mx = 0.f;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int ky = (int)(i % Wy);
    const float2 o = otf[i];
    const float2 m = otf[i - ky + (ky == 0 ? 0 : Wy - ky)];
    err = fmaxf(err, hypotf(o.x - m.x, o.y - m.y));
    mx = fmaxf(mx, hypotf(o.x, o.y));
  }
  for (int m = 16; m > 0; m >>= 1) {
    err = fmaxf(err, __shfl_xor_sync(0xffffffffu, err, m));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&bits[0], __float_as_uint(err));
    atomicMax(&bits[1], __float_as_uint(mx));
  }
}

// dst [Hx*Wz][owp] <- columns 0..Wy/2 of src [Hx*Wz][Wy] (pad column zero)
__global__ void otf_halve_kernel(const float2* __restrict__ src, float2* __restrict__ dst, size_t rows, int Wy,
                                 int owp) {
  const size_t n = rows * owp;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % owp);
    const size_t r = i / owp;
    dst[i] = c <= Wy / 2 ? src[r * Wy + c] : make_float2(0.f, 0.f);
  }
}

bool encode_otf_map(vk_rl_plan p, void* base, CUtensorMap* m);

// Replaces both full OTFs by their halves when both pass the mirror test
// (z pass with TMA OTF tiles only; VK_RL_NO_OTF_HALF=1 keeps the full ones).
void halve_otfs(vk_rl_plan p) {
  const char* no = std::getenv("VK_RL_NO_OTF_HALF");
  if ((no && no[0] == '1') || !p->otma || p->ofactored || p->g.Wy % 2) return;
  const Geom& g = p->g;
  DevBuf<unsigned> bits;
  bits.alloc(4, "otf check");
  ck(cudaMemsetAsync(bits.p, 0, 4 * sizeof(unsigned), p->stream), "otf check");
  const float2* o[2] = {p->otf.p, p->otf_flip.p};
  for (int k = 0; k < 2; ++k) {
    otf_mirror_check_kernel<<<148 * 8, 256, 0, p->stream>>>(o[k], g.Hx, g.Wz, g.Wy, bits.p + 2 * k);
    launch_check(p, "otf mirror check");
  }
  unsigned h[4];
  ck(cudaMemcpyAsync(h, bits.p, sizeof(h), cudaMemcpyDeviceToHost, p->stream), "otf check D2H");
  ck(cudaStreamSynchronize(p->stream), "otf check");
  for (int k = 0; k < 2; ++k) {
    float err, mx;
    std::memcpy(&err, &h[2 * k], 4);
    std::memcpy(&mx, &h[2 * k + 1], 4);
    if (!(mx > 0.f && err <= kOtfSepTol * mx)) return;
  }
  const int owp = (g.Wy / 2 + 2) / 2 * 2;
  const size_t rows = (size_t)g.Hx * g.Wz;
  DevBuf<float2> half[2];
  for (int k = 0; k < 2; ++k) {
    half[k].alloc(rows * owp, "half otf");
    otf_halve_kernel<<<148 * 8, 256, 0, p->stream>>>(o[k], half[k].p, rows, g.Wy, owp);
    launch_check(p, "otf halve");
  }
  ck(cudaStreamSynchronize(p->stream), "otf halve");
  std::swap(p->otf.p, half[0].p);
  std::swap(p->otf.n, half[0].n);
  std::swap(p->otf_flip.p, half[1].p);
  std::swap(p->otf_flip.n, half[1].n);  // the full tables are freed with half[]
  p->owp = owp;
  p->ohalf = true;
  if (!(encode_otf_map(p, p->otf.p, &p->omap) && encode_otf_map(p, p->otf_flip.p, &p->omap_flip)))
    fail(VK_ERR_CUDA, "half otf tensor map");
}

// Sets p->ofactored when both OTFs pass the rank-1 test (VK_RL_NO_OTF_FACTOR=1
// keeps the OTF reads).
void factor_otfs(vk_rl_plan p) {
  const char* no = std::getenv("VK_RL_NO_OTF_FACTOR");
  if (no && no[0] == '1') return;
  const Geom& g = p->g;
  const size_t nf = (size_t)g.Hx + g.Wy + g.Wz;
  p->ofac.alloc(2 * nf, "otf factors");
  DevBuf<unsigned> bits;
  bits.alloc(4, "otf check");
  ck(cudaMemsetAsync(bits.p, 0, 4 * sizeof(unsigned), p->stream), "otf check");
  const float2* o[2] = {p->otf.p, p->otf_flip.p};
  for (int k = 0; k < 2; ++k) {
    otf_factor_kernel<<<(unsigned)((nf + 255) / 256), 256, 0, p->stream>>>(o[k], g.Hx, g.Wz, g.Wy, p->ofac.p + k * nf);
    launch_check(p, "otf factor");
    otf_sep_check_kernel<<<148 * 8, 256, 0, p->stream>>>(o[k], p->ofac.p + k * nf, g.Hx, g.Wz, g.Wy, bits.p + 2 * k);
    launch_check(p, "otf separability");
  }
  unsigned h[4];
  ck(cudaMemcpyAsync(h, bits.p, sizeof(h), cudaMemcpyDeviceToHost, p->stream), "otf check D2H");
  ck(cudaStreamSynchronize(p->stream), "otf check");
  bool ok = true;
  for (int k = 0; k < 2; ++k) {
    float err, mx;
    std::memcpy(&err, &h[2 * k], 4);
    std::memcpy(&mx, &h[2 * k + 1], 4);
    ok = ok && mx > 0.f && err <= kOtfSepTol * mx;
  }
  p->ofactored = ok;
  if (!ok) p->ofac.free();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda):
// S_B as a 3D tensor {Wy, zrows, Hx} of 8-byte elements, box {16, Pz, 1}.
bool encode_zmap(vk_rl_plan p, int zrows, float2* base = nullptr, int planes = 0, CUtensorMap* out = nullptr) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return (EncodeFn)f;
  }();
  if (!fn) return false;
  const Geom& g = p->g;
  const cuuint64_t dims[3] = {(cuuint64_t)g.Wy, (cuuint64_t)zrows, (cuuint64_t)(planes ? planes : g.Hx)};
  const cuuint64_t strides[2] = {(cuuint64_t)g.Wy * 8, (cuuint64_t)zrows * g.Wy * 8};
  const cuuint32_t box[3] = {16, (cuuint32_t)g.Pz, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(out ? out : &p->zmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base ? base : p->SB.p, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// S_A [Hx][Pz][Py] as {Py, Pz, Hx}, box {2L rows, 1, tbk kx} for xpass_tma:
// nb = ceil(Hx / 256) boxes of tbk kx each, tbk a multiple of 128 / (16 L)
// so every box lands 128-byte aligned; the staged tile must fit the x tile.
bool encode_xmap(vk_rl_plan p) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return false;
  }
  const Geom& g = p->g;
  const int L = p->fx->Lx;
  if (g.Py % 2 || 2 * L > 256) return false;  // global strides must be multiples of 16 bytes
  const int nb = (g.Hx + 255) / 256, m = std::max(1, 128 / (16 * L));
  const int bk = ((g.Hx + nb - 1) / nb + m - 1) / m * m;
  if (bk > 256 || (size_t)nb * bk * 2 * L > (size_t)g.Wx * (L + 1)) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)g.Py, (cuuint64_t)g.Pz, (cuuint64_t)g.Hx};
  const cuuint64_t strides[2] = {(cuuint64_t)g.Py * 8, (cuuint64_t)g.Pz * g.Py * 8};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * L), 1, (cuuint32_t)bk};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (((EncodeFn)f)(&p->xmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, p->SA.p, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  p->xtbk = bk;
  p->xtnb = nb;
  return true;
}

// OTF [Hx][Wz][Wy] as {Wy, Wz, Hx}, box {16, Wz, 1}.
bool encode_otf_map(vk_rl_plan p, void* base, CUtensorMap* m) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return false;
  }
  const Geom& g = p->g;
  const cuuint64_t w = p->owp ? (cuuint64_t)p->owp : (cuuint64_t)g.Wy;  // half OTF: columns 0..owp-1
  const cuuint64_t dims[3] = {w, (cuuint64_t)g.Wz, (cuuint64_t)g.Hx};
  const cuuint64_t strides[2] = {w * 8, (cuuint64_t)g.Wz * w * 8};
  // half OTF: 18-column boxes (rl_fast.cuh kHalfBox: even, 16-byte aligned starts)
  const cuuint32_t box[3] = {p->owp ? 18u : 16u, (cuuint32_t)g.Wz, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return ((EncodeFn)f)(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Kernel attributes (dynamic shared memory, carveout) are per device
// context: set them once for every device a plan is created on.
cudaError_t fast_attributes_for_device(int device) {
  static std::mutex mu;
  static std::vector<int> done;  // 0 not yet, 1 ok
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0) return cudaErrorInvalidDevice;
  if ((int)done.size() <= device) done.resize(device + 1, 0);
  if (done[device]) return cudaSuccess;
  const cudaError_t e = vk::fast_init_attributes();  // on the current device (the caller's DeviceGuard)
  if (e == cudaSuccess) done[device] = 1;
  return e;
}

void to3(int rank, const uint64_t* in, uint64_t* out3) {
  for (int i = 0; i < 3; ++i) out3[i] = 1;
  for (int i = 0; i < rank; ++i) out3[3 - rank + i] = in[i];
}

// zslab (slab plans only): {P rows of the local domain, offset of the local
// image's first row inside it} for the z axis instead of I + 2 floor(K/2).
vk_rl_plan create_plan(int device, int rank, const uint64_t* shape, int psf_rank, const uint64_t* psf_shape,
                       const float* psf, int pad, int conv = 0, const int* zslab = nullptr) {
  if (rank < 1 || rank > VK_MAX_RANK) fail(VK_ERR_ARG, "rank must be 1, 2 or 3");
  if (psf_rank != rank)
    fail(VK_ERR_SHAPE, conv ? "ShapeMismatch: fft_convolve: rank mismatch"
                            : "ShapeMismatch: psf rank must match the image rank");
  if (conv == 2)  // filters.cpp:184-190
    for (int i = 0; i < rank; ++i)
      if (psf_shape[i] > shape[i])
        fail(VK_ERR_KERNEL_TOO_LARGE, "KernelTooLarge: circular convolution needs kernel <= image");
  for (int i = 0; i < rank; ++i) {
    if (shape[i] == 0) fail(VK_ERR_ARG, "empty image");
    if (psf_shape[i] == 0) fail(VK_ERR_ARG, "empty psf");
  }
  if (conv == 2) {
    // Circular convolution = the 'same' linear convolution of the periodic
    // extension, cropped (out[n] = sum_j k[j] a[(n + c - j) mod A], filters.cpp:
    // 184-233): the reference plans any extent with FFTW; the device FFT plans
    // 5-smooth grids, so any other extent goes through the linear path on
    // E = A + K - 1 with the image at offset h = K - 1 - c.
    bool smooth = true;
    for (int i = 0; i < rank; ++i) smooth = smooth && good_size(shape[i]) == shape[i];
    if (!smooth) {
      uint64_t E[VK_MAX_RANK];
      for (int i = 0; i < rank; ++i) E[i] = shape[i] + psf_shape[i] - 1;
      vk_rl_plan inner = create_plan(device, rank, E, psf_rank, psf_shape, psf, 0, 1);
      DeviceGuard dg(device);
      auto* p = new vk_rl_plan_s();
      p->device = device;
      p->rank = rank;
      p->pad = false;
      p->conv = 2;
      p->circ = inner;
      uint64_t I3[3], K3[3], E3[3];
      to3(rank, shape, I3);
      to3(rank, psf_shape, K3);
      to3(rank, E, E3);
      p->g = inner->g;
      p->g.Iz = (int)I3[0];
      p->g.Iy = (int)I3[1];
      p->g.Ix = (int)I3[2];
      for (int a = 0; a < 3; ++a) {
        p->circ_e[a] = (int)E3[a];
        p->circ_h[a] = (int)(K3[a] - 1 - (K3[a] - 1) / 2);
      }
      for (int i = 0; i < rank; ++i) {
        p->ishape[i] = shape[i];
        p->kshape[i] = psf_shape[i];
        p->dshape[i] = shape[i];
        p->wshape[i] = inner->wshape[i];
      }
      ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "cudaStreamCreate");
      return p;
    }
  }
  DeviceGuard dg(device);
  auto* p = new vk_rl_plan_s();
  try {
    p->device = device;
    p->rank = rank;
    p->pad = pad != 0;
    p->conv = conv;
    uint64_t I3[3], K3[3];
    to3(rank, shape, I3);
    to3(rank, psf_shape, K3);
    Geom& g = p->g;
    int* Ip[3] = {&g.Iz, &g.Iy, &g.Ix};
    int* Pp[3] = {&g.Pz, &g.Py, &g.Px};
    int* Op[3] = {&g.oz, &g.oy, &g.ox};
    int* Wp[3] = {&g.Wz, &g.Wy, &g.Wx};
    int* Cp[3] = {&g.cz, &g.cy, &g.cx};
    for (int a = 0; a < 3; ++a) {
      uint64_t off = p->pad ? K3[a] / 2 : 0;  // deconv.cpp:215-216
      uint64_t P = I3[a] + 2 * off;
      if (zslab && a == 0) {
        P = (uint64_t)zslab[0];
        off = (uint64_t)zslab[1];
      }
      // deconv.cpp:116 / filters.cpp:191-192; circular: the image grid itself
      uint64_t W = conv == 2 ? P : good_size(P + K3[a] - 1);
      if (zslab && a == 0) {
        // a slab's z grid is ours to choose (any W >= P+K-1 gives the same
        // linear correlation): the smallest compile-time fast length within
        // 1.5x of good_size, so the z pass keeps the register FFT
        for (uint64_t c = W; c <= W + W / 2; ++c)
          if (good_size(c) == c && vk::fast_lookup((int)c)) {
            W = c;
            break;
          }
      }
      if (P > (1u << 30) || W > (1u << 30)) fail(VK_ERR_ARG, "extent too large");
      if (good_size(W) != W)
        fail(VK_ERR_UNSUPPORTED, "circular fft_convolve on the B200 path needs 5-smooth extents (got " +
                                     std::to_string(W) + ")");
      *Ip[a] = (int)I3[a];
      *Pp[a] = (int)P;
      *Op[a] = (int)off;
      *Wp[a] = (int)W;
      *Cp[a] = conv == 2 ? 0 : (int)((K3[a] - 1) / 2);  // kernel_center, deconv.cpp:40
    }
    g.Hx = g.Wx / 2 + 1;
    p->Kz = (int)K3[0];
    p->Ky = (int)K3[1];
    p->Kx = (int)K3[2];
    for (int i = 0; i < rank; ++i) {
      p->ishape[i] = shape[i];
      p->kshape[i] = psf_shape[i];
    }
    p->psf_host.assign(psf, psf + (size_t)K3[0] * K3[1] * K3[2]);
    const uint64_t P3[3] = {(uint64_t)g.Pz, (uint64_t)g.Py, (uint64_t)g.Px};
    const uint64_t W3[3] = {(uint64_t)g.Wz, (uint64_t)g.Wy, (uint64_t)g.Wx};
    for (int i = 0; i < rank; ++i) {
      p->dshape[i] = P3[3 - rank + i];
      p->wshape[i] = W3[3 - rank + i];
    }

    // PSF value checks are stored and reported by runs in the reference's
    // order (deconv.cpp:319-326).
    size_t kn = (size_t)p->Kz * p->Ky * p->Kx;
    double sum = 0;
    for (size_t i = 0; i < kn; ++i) {
      if (psf[i] < 0) {
        p->psf_status = VK_ERR_NEGATIVE;
        p->psf_msg = "NegativeInput: psf must be nonnegative";
        break;
      }
      sum += psf[i];
    }
    if (p->psf_status == 0 && std::abs(sum - 1.0) > 1e-3) {
      p->psf_status = VK_ERR_UNNORMALIZED_PSF;
      p->psf_msg = "UnnormalizedPsf: psf sums to " + std::to_string(sum);
    }

    ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    auto tx = twiddles(g.Wx), ty = twiddles(g.Wy), tz = twiddles(g.Wz);
    p->twx.alloc(g.Wx, "twiddles");
    p->twy.alloc(g.Wy, "twiddles");
    p->twz.alloc(g.Wz, "twiddles");
    ck(cudaMemcpy(p->twx.p, tx.data(), tx.size() * sizeof(float2), cudaMemcpyHostToDevice), "twiddles");
    ck(cudaMemcpy(p->twy.p, ty.data(), ty.size() * sizeof(float2), cudaMemcpyHostToDevice), "twiddles");
    ck(cudaMemcpy(p->twz.p, tz.data(), tz.size() * sizeof(float2), cudaMemcpyHostToDevice), "twiddles");
    p->lpx = make_line_plan(g.Wx, p->twx.p);
    p->lpy = make_line_plan(g.Wy, p->twy.p);
    p->lpz = make_line_plan(g.Wz, p->twz.p);
    const char* gen = std::getenv("VK_RL_GENERIC");
    if (!(gen && gen[0] == '1')) {
      ck(fast_attributes_for_device(device), "fast kernel attributes");
      p->fx = vk::fast_lookup(g.Wx);
      p->fy = vk::fast_lookup(g.Wy);
      p->fz = g.Wz > 1 ? vk::fast_lookup(g.Wz) : nullptr;
      if (conv) p->fx = nullptr;  // XM_CONV_OUT lives in the generic x kernel
      if (p->fx) {  // butterfly-major pass-2 twiddles of the fast x pass (reg::load_twiddles2 layout)
        const auto t2 = fast_twiddles(p->fx, tx);
        p->twx2.alloc(t2.size(), "twiddles");
        ck(cudaMemcpy(p->twx2.p, t2.data(), t2.size() * sizeof(float2), cudaMemcpyHostToDevice), "twiddles");
        p->lpx.tw2 = p->twx2.p;
      }
      if (p->fz) {  // and the fast z pass
        const auto t2 = fast_twiddles(p->fz, tz);
        p->twz2.alloc(t2.size(), "twiddles");
        ck(cudaMemcpy(p->twz2.p, t2.data(), t2.size() * sizeof(float2), cudaMemcpyHostToDevice), "twiddles");
        p->lpz.tw2 = p->twz2.p;
      }
      if (p->fy) {  // same for the fast y pass
        const auto t2 = fast_twiddles(p->fy, ty);
        p->twy2.alloc(t2.size(), "twiddles");
        ck(cudaMemcpy(p->twy2.p, t2.data(), t2.size() * sizeof(float2), cudaMemcpyHostToDevice), "twiddles");
        p->lpy.tw2 = p->twy2.p;
      }
    }
    p->xL = pick_lines(g.Wx, 16, kSmemCap, x_smem);
    p->yL = pick_lines(g.Wy, 16, kSmemCap, yz_smem);
    p->zL = pick_lines(g.Wz, 16, kSmemCap, yz_smem);
    p->xs = x_smem(g.Wx, p->xL);
    p->ys = yz_smem(g.Wy, p->yL);
    p->zs = yz_smem(g.Wz, p->zL);
    constexpr size_t kMaxDyn = 227 * 1024 - 4096;  // leave room for static reduction scratch
    if (p->xs > kMaxDyn || p->ys > kMaxDyn || p->zs > kMaxDyn)
      fail(VK_ERR_UNSUPPORTED, "FFT length too large for the shared-memory line transform");
    ck(cudaFuncSetAttribute(vk::xpass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDyn),
       "smem attr");
    ck(cudaFuncSetAttribute(vk::ypass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDyn),
       "smem attr");
    ck(cudaFuncSetAttribute(vk::zpass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDyn),
       "smem attr");

    const char* noyt = std::getenv("VK_RL_NO_YTMA");
    const char* notma0 = std::getenv("VK_RL_NO_TMA");
    p->ytma = p->fy && p->fy->ytk && !(notma0 && notma0[0] == '1') && !(noyt && noyt[0] == '1');
    const size_t sa = (size_t)g.Hx * std::max(g.Pz, p->Kz) * std::max(g.Py, p->Ky);
    const size_t sb = (size_t)g.Hx * std::max(g.Pz, p->Kz) * g.Wy;
    const size_t so = (size_t)g.Hx * g.Wz * g.Wy;
    // the pass kernels index spectra and the padded domain with 32-bit offsets
    if (so >= (1ull << 32) || sb >= (1ull << 32) || (size_t)g.Pz * g.Py * g.Px >= (1ull << 32))
      fail(VK_ERR_UNSUPPORTED, "volume too large for one plan (spectrum >= 2^32 elements): split it into slabs "
                               "(vk_rl_slab_plan_create)");
    p->SA.alloc(sa, "spectrum A");
    // TMA-staged x passes (xpass_tma) wherever the fast x pass runs and S_A's
    // rows are 16-byte multiples; VK_RL_NO_XTMA=1 keeps the per-thread loads
    if (p->fx && p->fx->xtk) {
      const char* nx = std::getenv("VK_RL_NO_XTMA");
      p->xtma = !(nx && nx[0] == '1') && encode_xmap(p);
    }
    if (g.Wz > 1) p->SB.alloc(sb, "spectrum B");
    // TMA-staged z tile (zpass_tma) where the length has one and the box
    // fits (Pz <= 256): C2 z convolutions 0.313 vs 0.345 ms per iteration
    // with cp.async (profiles/r01/final/tma.log).  VK_RL_NO_TMA=1 disables.
    const char* notma = std::getenv("VK_RL_NO_TMA");
    // x-pass L2 prefetch of the CTA's spectrum chunks and observed/estimate
    // rows at entry, for 3D grids: C2 -4.1%, C4 -5.9%, C1 -1.6% per
    // iteration; 2D fields +3% (profiles/r01/final/xpf.log).  VK_RL_XPF=mask
    // overrides (1 spectrum, 2 rows).
    p->xpf = g.Wz > 1 ? 3 : 0;
    if (const char* nts = std::getenv("VK_RL_NO_TMA_STORE")) p->tma_store = nts[0] != '1';
    if (const char* xpf = std::getenv("VK_RL_XPF")) p->xpf = std::atoi(xpf);
    if (p->fz && p->fz->ztk && g.Wz > 1 && g.Pz <= 256 && g.Wy % 2 == 0 && !(notma && notma[0] == '1'))
      p->ztma = encode_zmap(p, std::max(g.Pz, p->Kz));
    // kx-chunked y/z convolution where S_B does not fit L2 anyway (> 64 MB);
    // small volumes (C1/C3, S_B 26 MB) keep the whole-volume passes.  Chunk
    // count: a multiple of the stream count (the streams' last chunks end
    // together: C4 +1.0%) near Hx * ceil(Wy/16) / T z-tile CTAs per chunk,
    // T = 1250 on 2 streams (C2: 8 chunks, 3.72e10 vs 3.69e10 / 3.60e10 at
    // 10 / 6; C4: 30 chunks, 3.589e10 vs 3.571e10 / 3.557e10 at 38 / 24) and
    // 650 on 3 (C2 15 chunks: +0.4 to +1.0% over 2 streams; C4 57: equal):
    // profiles/r02/kxchunk_even_ab.txt.  3 streams by default.
    // VK_RL_KXCHUNK = target MB of S_B per chunk instead (0 = whole volume).
    if (p->ztma && !conv && !zslab) {
      const char* kc = std::getenv("VK_RL_KXCHUNK");
      if (const char* ks = std::getenv("VK_RL_KXSTREAMS")) p->kxs = std::max(2, std::min(4, std::atoi(ks)));
      const double sb_mb = (double)g.Hx * g.Pz * g.Wy * 8 / 1e6;
      int nch = 0;
      if (kc) {
        const double mb = std::atof(kc);
        if (mb > 0) {
          const int c = std::max(1, (int)(mb * 1e6 / ((double)g.Pz * g.Wy * 8)));
          nch = (g.Hx + c - 1) / c;
        }
      } else if (sb_mb > 64.0) {
        // z-tile CTAs per chunk: 1250 on 2 streams, 650 on 3 (C2 sweep:
        // 15 chunks of 19 planes on 3 streams), 500 on 4
        const double per = p->kxs == 2 ? 1250.0 : p->kxs == 3 ? 650.0 : 500.0;
        nch = (int)std::lround((double)g.Hx * ((g.Wy + 15) / 16) / per);
        // at most 64 chunks: the paper's 90x6480x7680 grid would otherwise
        // get 2394 chunks of 2 planes (5.57e8 vs 6.03e8 voxel-iters/s with 60,
        // profiles/r02/paper_volume.md)
        nch = std::min(nch, 64);
      }
      if (nch > 1) {
        nch = std::max(p->kxs, (int)std::lround((double)nch / p->kxs) * p->kxs);
        nch = std::min(nch, g.Hx);  // no empty chunk
        p->kxn = nch;
        p->kxc = (g.Hx + nch - 1) / nch;  // ring slot: the largest chunk
      }
      if (p->kxc) {
        p->ring2.alloc((size_t)p->kxs * p->kxc * g.Pz * g.Wy, "S_B ring");
        for (int k = 0; k < p->kxs; ++k)
          if (!encode_zmap(p, g.Pz, p->ring2.p + (size_t)k * p->kxc * g.Pz * g.Wy, p->kxc, &p->zmap_ring[k]))
            p->kxc = 0;
        const char* pe = std::getenv("VK_RL_RING_PERSIST");
        int dev = 0, max_persist = 0, max_window = 0;
        if (p->kxc && pe && pe[0] == '1' && cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev) == cudaSuccess &&
            max_persist > 0 && max_window > 0) {
          const size_t bytes = p->ring2.n * sizeof(float2);
          size_t cur = 0;
          cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
          if (cur < std::min(bytes, (size_t)max_persist))
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(bytes, (size_t)max_persist));
          p->ring_window = std::min(bytes, (size_t)max_window);
        }
        cudaGetLastError();
      }
    }
    p->otf.alloc(so, "otf");
    if (!conv) p->otf_flip.alloc(so, "otf_flip");
    if (p->ztma && !conv && g.Wz <= 256) {  // OTF tiles by TMA too (VK_RL_NO_OTF_TMA=1 disables)
      const char* no = std::getenv("VK_RL_NO_OTF_TMA");
      p->otma = !(no && no[0] == '1') && encode_otf_map(p, p->otf.p, &p->omap) &&
                encode_otf_map(p, p->otf_flip.p, &p->omap_flip);
    }
    p->est.alloc((size_t)g.Pz * g.Py * g.Px, "estimate");
    p->stats.alloc(1, "stats");
    p->ycrop = g.cy;  // until the OTF ramp below folds it in

    // Both spectra: psf and std::reverse(psf) == flip about every axis.
    std::vector<float> flipped(psf, psf + kn);
    std::reverse(flipped.begin(), flipped.end());
    DevBuf<float> dpsf;
    dpsf.alloc(kn, "psf");
    ck(cudaMemcpyAsync(dpsf.p, psf, kn * sizeof(float), cudaMemcpyHostToDevice, p->stream), "psf H2D");
    if (conv == 2) {  // circular: centre-wrapped kernel on the full grid
      DevBuf<float> wrapped;
      const size_t wn = (size_t)g.Wz * g.Wy * g.Wx;
      wrapped.alloc(wn, "wrapped kernel");
      ck(cudaMemsetAsync(wrapped.p, 0, wn * sizeof(float), p->stream), "wrap");
      vk::wrap_kernel_kernel<<<148, kThreads, 0, p->stream>>>(dpsf.p, p->Kz, p->Ky, p->Kx, g.Wz, g.Wy, g.Wx,
                                                               wrapped.p);
      launch_check(p, "wrap kernel");
      spectrum3d(p, p->stream, wrapped.p, g.Wz, g.Wy, g.Wx,
                 (float)(1.0 / ((double)g.Wz * g.Wy * g.Wx)), p->otf.p);
      ck(cudaStreamSynchronize(p->stream), "otf");
      p->launches = 0;
      return p;
    }
    build_otf(p, dpsf.p, p->otf.p);
    if (conv) {
      ck(cudaStreamSynchronize(p->stream), "otf");
      p->launches = 0;
      return p;
    }
    ck(cudaStreamSynchronize(p->stream), "otf");
    ck(cudaMemcpyAsync(dpsf.p, flipped.data(), kn * sizeof(float), cudaMemcpyHostToDevice, p->stream),
       "psf H2D");
    build_otf(p, dpsf.p, p->otf_flip.p);
    // The fast x-pass keeps rows at [cx, cx+Px): the x crop is a phase ramp.
    // Where the y inverse bulk-stores its lines (ypass_tma), the y crop is one
    // too, so the cropped lines start at slot 0 (16-byte aligned); C2 y inverse
    // -10% (profiles/r01/final/tst.log).
    const bool yramp = p->fy && p->ytma && p->tma_store && g.cy != 0;
    p->ycrop = yramp ? 0 : g.cy;
    const int cxr = p->fx ? g.cx : 0, cyr = yramp ? g.cy : 0;
    if (cxr != 0 || cyr != 0) {
      const size_t plane = (size_t)g.Wz * g.Wy;
      ck(vk::launch_otf_ramp(p->otf.p, g.Hx, plane, g.Wx, cxr, g.Wy, cyr, p->stream), "otf ramp");
      ck(vk::launch_otf_ramp(p->otf_flip.p, g.Hx, plane, g.Wx, cxr, g.Wy, cyr, p->stream), "otf ramp");
    }
    ck(cudaStreamSynchronize(p->stream), "otf_flip");
    if (p->ztma || (g.Wz == 1 && p->fy && p->ytma)) factor_otfs(p);
    // richardson_lucy plans only: the FRC sub-plan (pad = 0) uses its OTF
    // buffers as full-size spectrum scratch
    if (p->ztma && !conv && p->pad) halve_otfs(p);
    p->launches = 0;
  } catch (...) {
    delete p;
    throw;
  }
  return p;
}

void ensure_iter_buffers(vk_rl_plan p, int iters) {
  p->sum_done = 0;
  if (!p->part.p) p->part.alloc((size_t)kStatBlocks * 8, "block partials");
  if (!p->xpart.p) {  // x-pass grid: ceil(Py / 2L) x Pz blocks (x_pass)
    const int L = p->fx ? p->fx->Lx : p->xL;
    p->xblocks = (p->g.Py + 2 * L - 1) / (2 * L) * p->g.Pz;
    p->xpart.alloc((size_t)kSumRing * p->xblocks * 4, "x-pass partials");
  }
  if (iters <= p->acc_cap) return;
  p->acc.alloc((size_t)iters * 4, "trace accumulators");
  if (p->h_acc) cudaFreeHost(p->h_acc);
  p->h_acc = nullptr;
  ck(cudaMallocHost(&p->h_acc, (size_t)iters * 4 * sizeof(double)), "pinned trace");
  while ((int)p->events.size() < iters + 1) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event");
    p->events.push_back(e);
  }
  p->acc_cap = iters;
}

void check_rule(const vk_stop_rule* r) {
  if (!r) fail(VK_ERR_ARG, "rule is NULL");
  if (r->rel_tol <= 0 && !std::isinf(r->rel_tol)) fail(VK_ERR_ARG, "rel_tol must be positive");
  if (r->patience < 1) fail(VK_ERR_ARG, "patience must be >= 1");
  if (r->max_iters < 1) fail(VK_ERR_ARG, "max_iters must be >= 1");
}

double relative_change(double prev, double cur) {  // deconv.cpp:296-300
  if (std::isinf(prev) && std::isinf(cur) && prev == cur) return 0.0;
  if (std::isinf(prev) || std::isinf(cur)) return std::numeric_limits<double>::infinity();
  return std::abs(cur - prev) / std::max(std::abs(prev), 1e-30);
}

// Replays the stopping rule over metric values 1..n (deconv.cpp:409-423):
// from iteration 2 on, a relative change below rel_tol counts a failure,
// anything else resets; patience failures in a row stop the run.
bool rule_fires(const std::vector<double>& values, int n, const vk_stop_rule* rule) {
  int fails = 0;
  for (int k = 1; k < n; ++k) {
    fails = relative_change(values[k - 1], values[k]) < rule->rel_tol ? fails + 1 : 0;
    if (fails >= rule->patience) return true;
  }
  return false;
}

struct RefStats {
  double n, sr, srr, range;
};

// si_psnr(current, observed) from fused sums (metrics.cpp:67-101).  The
// residual uses the least-squares identity mean((a x + b - r)^2) =
// var_r - a cov(x, r), exact in exact arithmetic.
double si_psnr_from_sums(const RefStats& r, double sx, double sxx, double sxr) {
  const double n = r.n;
  const double var_r = r.srr / n - (r.sr / n) * (r.sr / n);
  if (var_r <= 0.0) fail(VK_ERR_DEGENERATE_REF, "DegenerateReference: si_psnr needs a non-constant reference");
  const double var_x = sxx / n - (sx / n) * (sx / n);
  const double cov = sxr / n - (sx / n) * (r.sr / n);
  double a = 0.0;
  if (var_x > 0.0) a = cov / var_x;
  const double err = var_r - a * cov;
  if (err <= 0.0) return std::numeric_limits<double>::infinity();
  return 10.0 * std::log10(r.range * r.range / err);
}

// Sub-plan and buffers for single_image_frc of the image crop
// (metrics.cpp:241-264): even_view trims odd extents, the half extents must be
// 5-smooth for the device r2c (no Bluestein yet).
void setup_frc(vk_rl_plan p) {
  if (p->frc || p->frc_dft) return;
  uint64_t half[3] = {1, 1, 1}, ones[3] = {1, 1, 1};
  bool smooth = true;
  for (int a = 0; a < p->rank; ++a) {
    const uint64_t e = p->ishape[a] - p->ishape[a] % 2;  // even_view (deconv.cpp:255-276)
    if (e == 0) fail(VK_ERR_UNSUPPORTED, "frc_resolution needs every image extent >= 2");
    half[a] = e / 2;
    smooth = smooth && good_size(half[a]) == half[a];
  }
  const float one = 1.0f;
  if (smooth) p->frc = create_plan(p->device, p->rank, half, p->rank, ones, &one, 0);
  p->frc_dft = !smooth;
  uint64_t nmax = 0;
  for (int a = 0; a < p->rank; ++a) nmax = std::max(nmax, half[a]);
  p->frc_binf = 1.0 / (double)nmax;  // ring_width / n_max (metrics.cpp:166-169)
  p->frc_nbins = (int)std::floor(0.5 / p->frc_binf) + 1;
  if ((double)p->ishape[0] * p->ishape[p->rank > 1 ? 1 : 0] * 2 > 2e9)
    fail(VK_ERR_UNSUPPORTED, "frc_resolution: image too large for the ring-sum kernel");
  {  // per-warp ring histograms while they fit in shared memory, else fewer
    const size_t one = (size_t)3 * p->frc_nbins * sizeof(double);
    int sl = kThreads / 32;
    while (sl > 1 && one * sl > 96 * 1024) sl >>= 1;
    p->frc_slices = sl;
    if (one * sl > 200 * 1024) fail(VK_ERR_UNSUPPORTED, "frc_resolution: image too large for the ring histogram");
    ck(cudaFuncSetAttribute(vk::frc_bins_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(one * sl)),
       "frc smem");
  }
  for (int a3 = 0; a3 < 3; ++a3) {
    const int a = a3 - (3 - p->rank);
    p->frc_h[a3] = a >= 0 ? (int)half[a] : 1;
    p->frc_s[a3] = a >= 0 ? 1 : 0;
  }
  const size_t hn = (size_t)p->frc_h[0] * p->frc_h[1] * p->frc_h[2];
  p->frc_even.alloc(hn, "frc even");
  p->frc_odd.alloc(hn, "frc odd");
  if (p->frc_dft) {
    const size_t cn = (size_t)p->frc_h[0] * p->frc_h[1] * (p->frc_h[2] / 2 + 1);
    p->frc_t1.alloc(2 * cn, "frc dft scratch");
    p->frc_A.alloc(cn, "frc spectrum A");
    p->frc_B.alloc(cn, "frc spectrum B");
    for (int a = 0; a < 3; ++a) {  // exp(-2 pi i m / n), m < n, from the exact angle
      const int n = p->frc_h[a];
      std::vector<float2> tw(n);
      for (int m = 0; m < n; ++m) {
        const double ang = -2.0 * M_PI * (double)m / (double)n;
        tw[m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
      p->frc_tw[a].alloc(n, "frc twiddles");
      ck(cudaMemcpy(p->frc_tw[a].p, tw.data(), n * sizeof(float2), cudaMemcpyHostToDevice), "frc twiddles");
    }
  }
  p->frc_bins.alloc((size_t)3 * p->frc_nbins * (1 + kFrcBlocks), "frc bins");  // [sums | per-block partials]
  ck(cudaMallocHost(&p->h_frc, (size_t)3 * p->frc_nbins * sizeof(double)), "frc pinned");
}

// frc_resolution(frc(even, odd), 2*spacing) of the current estimate crop
// (metrics.cpp:146-239): the ring sums into frc_bins (no sync).
void frc_bins_enqueue(vk_rl_plan p, cudaStream_t s) {
  vk_rl_plan_s* f = p->frc;
  const int nb = p->frc_nbins;

  vk::frc_split_kernel<<<148 * 4, kThreads, 0, s>>>(p->est.p, p->g, p->frc_h[0], p->frc_h[1], p->frc_h[2],
                                                     p->frc_s[0], p->frc_s[1], p->frc_s[2], p->frc_even.p,
                                                     p->frc_odd.p);
  launch_check(p, "frc split");
  if (p->frc_dft) {
    // r2c along x, then y, then z (written in the [Hx][hz][hy] bins layout)
    const int hz = p->frc_h[0], hy = p->frc_h[1], hx = p->frc_h[2], Hx = hx / 2 + 1;
    const long long cy = Hx, cz = (long long)hy * Hx;
    float2* t1 = p->frc_t1.p;
    float2* t2 = p->frc_t1.p + (size_t)hz * hy * Hx;
    const int grid = 148 * 8;
    for (int img = 0; img < 2; ++img) {
      const float* src = img ? p->frc_odd.p : p->frc_even.p;
      float2* dst = img ? p->frc_B.p : p->frc_A.p;
      vk::dft_axis_kernel<true><<<grid, kThreads, 0, s>>>(src, t1, hz, hy, Hx, 2, hx, (long long)hy * hx, hx, 1,
                                                          cz, cy, 1, p->frc_tw[2].p);
      vk::dft_axis_kernel<false><<<grid, kThreads, 0, s>>>(t1, t2, hz, hy, Hx, 1, hy, cz, cy, 1, cz, cy, 1,
                                                           p->frc_tw[1].p);
      vk::dft_axis_kernel<false><<<grid, kThreads, 0, s>>>(t2, dst, hz, hy, Hx, 0, hz, cz, cy, 1, hy, 1,
                                                           (long long)hz * hy, p->frc_tw[0].p);
      launch_check(p, "frc dft");
    }
    vk::frc_bins_kernel<<<kFrcBlocks, kThreads, (size_t)3 * nb * p->frc_slices * sizeof(double), s>>>(
        p->frc_A.p, p->frc_B.p, hz, hy, hx, Hx, p->frc_binf, nb, p->frc_bins.p + 3 * nb, p->frc_slices);
    launch_check(p, "frc bins");
  } else {
    const vk::Geom& fg = f->g;
    spectrum3d(f, s, p->frc_even.p, fg.Pz, fg.Py, fg.Px, 1.0f, f->otf.p);
    spectrum3d(f, s, p->frc_odd.p, fg.Pz, fg.Py, fg.Px, 1.0f, f->otf_flip.p);
    vk::frc_bins_kernel<<<kFrcBlocks, kThreads, (size_t)3 * nb * p->frc_slices * sizeof(double), s>>>(
        f->otf.p, f->otf_flip.p, fg.Wz, fg.Wy, fg.Wx, fg.Hx, p->frc_binf, nb, p->frc_bins.p + 3 * nb,
        p->frc_slices);
    launch_check(p, "frc bins");
  }
  vk::frc_bins_reduce<<<3 * nb, 256, 0, s>>>(p->frc_bins.p + 3 * nb, kFrcBlocks, 3 * nb, p->frc_bins.p);
  launch_check(p, "frc reduce");
}

// ... and the host walks the few hundred ring values (one sync).
double frc_eval(vk_rl_plan p, cudaStream_t s, double spacing) {
  frc_bins_enqueue(p, s);
  const int nb = p->frc_nbins;
  ck(cudaMemcpyAsync(p->h_frc, p->frc_bins.p, (size_t)3 * nb * sizeof(double), cudaMemcpyDeviceToHost, s),
     "frc D2H");
  ck(cudaStreamSynchronize(s), "frc");
  const double* num = p->h_frc;
  const double* da = p->h_frc + nb;
  const double* db = p->h_frc + 2 * nb;
  auto corr = [&](int j) {
    const double den = std::sqrt(da[j] * db[j]);
    return den > 0 ? num[j] / den : 0.0;
  };
  const double threshold = 1.0 / 7.0, sp = spacing * 2.0;  // single_image_frc doubles the spacing
  for (int j = 1; j < nb; ++j) {  // DC excluded (metrics.cpp:221-239)
    if (corr(j) < threshold) {
      double nu;
      if (j == 1 || corr(j - 1) < threshold) {
        nu = j * p->frc_binf;
      } else {
        const double c0 = corr(j - 1), c1 = corr(j);
        const double f0 = (j - 1) * p->frc_binf, f1 = j * p->frc_binf;
        nu = f0 + (f1 - f0) * (c0 - threshold) / (c0 - c1);
      }
      if (nu <= 0) return std::numeric_limits<double>::infinity();
      return sp / nu;
    }
  }
  return std::numeric_limits<double>::infinity();  // kUnresolved
}

// Buffers for ssim_vs_prev (metrics.cpp:103-144): TooSmall below 7 voxels
// per axis (raised at the first metric evaluation in the reference, before
// any estimate is returned either way).
void setup_ssim(vk_rl_plan p, int iters) {
  for (int a = 0; a < p->rank; ++a)
    if (p->ishape[a] < 7) fail(VK_ERR_TOO_SMALL, "ssim needs every extent >= 7");
  const Geom& g = p->g;
  const size_t nI = (size_t)g.Iz * g.Iy * g.Ix;
  if (!p->ss_ready) {
    for (auto& b : p->ss_img) b.alloc(nI, "ssim images");
    for (int k = 0; k < std::min(p->rank - 1, 2); ++k) p->ss_f[k].alloc(5 * nI, "ssim moments");
    p->ss_ready = true;
  }
  if (iters > p->ss_cap) {
    p->ss_range.alloc((size_t)(iters + 1) * 2, "ssim ranges");
    p->ss_sum.alloc((size_t)iters, "ssim sums");
    p->ss_cap = iters;
  }
}

// The three separable smoothing passes and the SSIM-map sum of cur against
// prev (whose range is range_prev[0..1]), reduced in a fixed order into *sum.
void ssim_passes(vk_rl_plan p, cudaStream_t s, const float* cur, const float* prev, const unsigned* range_prev,
                 double* sum_out) {
  const Geom& g = p->g;
  const size_t nI = (size_t)g.Iz * g.Iy * g.Ix;
  static const vk::SsimTaps taps = [] {  // filters.cpp:78-90
    vk::SsimTaps t{};
    const double sigma = 1.5;
    double sum = 0;
    for (int i = -vk::kSsimHalf; i <= vk::kSsimHalf; ++i) {
      const double v = std::exp(-0.5 * (i / sigma) * (i / sigma));
      t.w[i + vk::kSsimHalf] = v;
      sum += v;
    }
    for (double& v : t.w) v /= sum;
    return t;
  }();
  double* sum = p->part.p;  // block partials of the last pass
  const int grid = 148 * 8;
  size_t stride = 1;
  size_t strides[3];
  for (int a = p->rank - 1; a >= 0; --a) {
    strides[a] = stride;
    stride *= p->ishape[a];
  }
  const unsigned* range = range_prev;
  for (int k = 0; k < p->rank; ++k) {
    const int ext = (int)p->ishape[k];
    const double* in = k == 0 ? nullptr : p->ss_f[(k - 1) % 2].p;
    double* out = k == p->rank - 1 ? nullptr : p->ss_f[k % 2].p;
    const bool first = k == 0, last = k == p->rank - 1;
    if (first && last)
      vk::ssim_axis_kernel<true, true><<<grid, kThreads, 0, s>>>(cur, prev, in, out, nI, ext, strides[k], taps,
                                                                   range, sum);
    else if (first)
      vk::ssim_axis_kernel<true, false><<<grid, kThreads, 0, s>>>(cur, prev, in, out, nI, ext, strides[k], taps,
                                                                    range, sum);
    else if (last)
      vk::ssim_axis_kernel<false, true><<<grid, kThreads, 0, s>>>(cur, prev, in, out, nI, ext, strides[k], taps,
                                                                    range, sum);
    else
      vk::ssim_axis_kernel<false, false><<<grid, kThreads, 0, s>>>(cur, prev, in, out, nI, ext, strides[k],
                                                                     taps, range, sum);
    launch_check(p, "ssim pass");
  }
  vk::reduce_partials_kernel<<<1, 256, 0, s>>>(p->part.p, grid, 1, sum_out);
  launch_check(p, "ssim reduce");
}

// ssim(crop(est), previous) for iteration `it` (1-based); previous is the
// observed image at it = 1 and the crop of iteration it-1 afterwards
// (deconv.cpp:352, 403, 423).  The sum lands in ss_sum[it-1]; no sync.
void ssim_eval(vk_rl_plan p, cudaStream_t s, int it, const float* d_obs) {
  const Geom& g = p->g;
  float* cur = p->ss_img[it % 2].p;
  const float* prev = it == 1 ? d_obs : p->ss_img[(it - 1) % 2].p;
  vk::crop_range_kernel<<<148 * 4, kThreads, 0, s>>>(p->est.p, cur, g, p->ss_range.p + 2 * it);
  launch_check(p, "ssim crop");
  ssim_passes(p, s, cur, prev, p->ss_range.p + 2 * (it - 1), p->ss_sum.p + (it - 1));
}

// ssim_vs_prev inside the graph body: fixed slots instead of the per-iteration
// ping-pong -- current crop ss_img[0] and range row 1, previous ss_img[1] and
// row 0 (seeded with the observed image), rolled over after the evaluation;
// the SSIM-map sum lands in gmetric.
void ssim_eval_graph(vk_rl_plan p, cudaStream_t s) {
  const Geom& g = p->g;
  const size_t nI = (size_t)g.Iz * g.Iy * g.Ix;
  ck(cudaMemcpyAsync(p->ss_range.p + 2, p->grange_init.p, 2 * sizeof(unsigned), cudaMemcpyDeviceToDevice, s),
     "ssim range");
  vk::crop_range_kernel<<<148 * 4, kThreads, 0, s>>>(p->est.p, p->ss_img[0].p, g, p->ss_range.p + 2);
  launch_check(p, "ssim crop");
  ssim_passes(p, s, p->ss_img[0].p, p->ss_img[1].p, p->ss_range.p, p->gmetric.p);
  ck(cudaMemcpyAsync(p->ss_img[1].p, p->ss_img[0].p, nI * sizeof(float), cudaMemcpyDeviceToDevice, s), "ssim roll");
  ck(cudaMemcpyAsync(p->ss_range.p, p->ss_range.p + 2, 2 * sizeof(unsigned), cudaMemcpyDeviceToDevice, s),
     "ssim roll");
}

// Iterations 1.. of richardson_lucy with the stopping rule decided on the
// device (deconv.cpp:401-423): one iteration = one CUDA graph (convolutions,
// x passes, metric, rule kernel) under a WHILE conditional node; the rule
// kernel sets the condition, so nothing returns to the host until the run
// ends.  The graph is built once per (observed buffer, rule) and replayed.
// Outputs: iterations run, stop flag, per-iteration metric values, device
// timestamps (wall_s), and acc rows (LL, sums).
void run_graph_loop(vk_rl_plan p, cudaStream_t s, const float* d_obs, const vk_stop_rule* rule, bool frc, bool ssim,
                    double spacing, std::vector<double>& values, std::vector<double>& wall, int& run, bool& stopped) {
  const Geom& g = p->g;
  const int iters = rule->max_iters;
  const size_t nI = (size_t)g.Iz * g.Iy * g.Ix;
  if (!p->gstate.p) {
    p->gstate.alloc(1, "stop state");
    p->gmetric.alloc(1, "metric");
    p->grange_init.alloc(2, "range init");
    const unsigned init[2] = {0x7f800000u, 0u};
    ck(cudaMemcpy(p->grange_init.p, init, sizeof(init), cudaMemcpyHostToDevice), "range init");
  }
  if (p->gvalues.n < (size_t)iters) {
    p->gvalues.alloc(iters, "metric values");
    p->gts.alloc(iters + 1, "timestamps");
  }
  const int metric = frc ? VK_METRIC_FRC_RESOLUTION : ssim ? VK_METRIC_SSIM_VS_PREV : VK_METRIC_SI_PSNR_VS_INPUT;
  vk_rl_plan_s::GraphKey key;
  key.obs = d_obs;
  key.metric = metric;
  key.iters = iters;
  key.patience = rule->patience;
  key.rel_tol = rule->rel_tol;
  key.spacing = spacing;
  if (!p->grx || !(key == p->grkey)) {
    if (p->grx) cudaGraphExecDestroy(p->grx);
    if (p->gr) cudaGraphDestroy(p->gr);
    p->grx = nullptr;
    p->gr = nullptr;
    ck(cudaGraphCreate(&p->gr, 0), "graph");
    cudaGraphConditionalHandle h;
    ck(cudaGraphConditionalHandleCreate(&h, p->gr, 1, cudaGraphCondAssignDefault), "graph condition");
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    ck(cudaGraphAddNode(&node, p->gr, nullptr, 0, &cp), "graph while node");
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    const uint64_t before = p->launches;
    // The body is captured on the plan's own stream: the caller's `s` may be
    // the legacy NULL stream, which cannot capture.  Only the launch uses `s`.
    cudaStream_t cs = p->stream;
    ck(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal), "capture");
    t_capturing = true;
    try {
      conv_yz(p, cs, p->otf.p);
      // every iteration's partials in slot 0: the rule kernel reduces them before the next
      x_pass(p, cs, vk::XM_RATIO, nullptr, g.Pz, g.Py, g.Px, 1.f, p->est.p, d_obs, 1, nullptr);
      conv_yz(p, cs, p->otf_flip.p);
      x_pass(p, cs, vk::XM_UPDATE, nullptr, g.Pz, g.Py, g.Px, 1.f, p->est.p, d_obs, 1, nullptr);
      if (frc) {
        frc_bins_enqueue(p, cs);
        vk::frc_value_kernel<<<1, 32, 0, cs>>>(p->frc_bins.p, p->frc_nbins, p->frc_binf, spacing, p->gmetric.p);
        launch_check(p, "frc value");
      }
      if (ssim) ssim_eval_graph(p, cs);
      vk::RuleArgs ra{};
      ra.st = p->gstate.p;
      ra.values = p->gvalues.p;
      ra.ts = p->gts.p;
      ra.xpart = p->xpart.p;
      ra.nblocks = p->xblocks;
      ra.acc = p->acc.p;
      ra.obs = p->stats.p;
      ra.n_img = (double)nI;
      ra.metric_in = p->gmetric.p;
      ra.metric = metric;
      ra.rel_tol = rule->rel_tol;
      ra.patience = rule->patience;
      ra.iters = iters;
      ra.handle = h;
      vk::rule_step_kernel<<<1, 256, 0, cs>>>(ra);
      launch_check(p, "rule");
    } catch (...) {
      t_capturing = false;
      cudaGraph_t junk;
      cudaStreamEndCapture(cs, &junk);
      cudaGetLastError();
      throw;
    }
    t_capturing = false;
    ck(cudaStreamEndCapture(cs, &body), "end capture");
    ck(cudaGraphInstantiate(&p->grx, p->gr, 0), "graph instantiate");
    p->gr_body_launches = p->launches - before;
    p->launches = before;
    p->grkey = key;
  }
  ck(cudaMemsetAsync(p->gstate.p, 0, sizeof(vk::StopState), s), "stop state");
  vk::timestamp_kernel<<<1, 1, 0, s>>>(p->gts.p);
  launch_check(p, "timestamp");
  if (ssim) {  // previous = the observed image (deconv.cpp:352), its range already in row 0
    ck(cudaMemcpyAsync(p->ss_img[1].p, d_obs, nI * sizeof(float), cudaMemcpyDeviceToDevice, s), "ssim seed");
  }
  ck(cudaGraphLaunch(p->grx, s), "graph launch");
  vk::StopState st{};
  ck(cudaMemcpyAsync(&st, p->gstate.p, sizeof(st), cudaMemcpyDeviceToHost, s), "stop state D2H");
  ck(cudaStreamSynchronize(s), "graph run");
  run = st.it;
  stopped = st.stopped != 0;
  p->launches += p->gr_body_launches * (uint64_t)run;
  values.resize(run);
  std::vector<unsigned long long> ts(run + 1);
  ck(cudaMemcpy(values.data(), p->gvalues.p, run * sizeof(double), cudaMemcpyDeviceToHost), "values D2H");
  ck(cudaMemcpy(ts.data(), p->gts.p, (run + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "ts D2H");
  wall.resize(run);
  for (int k = 0; k < run; ++k) wall[k] = (double)(ts[k + 1] - ts[k]) * 1e-9;
  p->sum_done = run;  // acc rows were written by the rule kernel
}

// The richardson_lucy loop on device buffers (deconv.cpp:333-430).
void run_device(vk_rl_plan p, const float* d_obs, float* d_out, const vk_stop_rule* rule, int flat_init,
                vk_trace* trace, cudaStream_t s, bool check_obs) {
  check_rule(rule);
  if (p->conv) fail(VK_ERR_ARG, "plan was created for fft_convolve");
  if (!p->pad) fail(VK_ERR_ARG, "plan was created without padding (rl_step plan)");
  if (rule->metric != VK_METRIC_SI_PSNR_VS_INPUT && rule->metric != VK_METRIC_FRC_RESOLUTION &&
      rule->metric != VK_METRIC_SSIM_VS_PREV)
    fail(VK_ERR_ARG, "unknown stopping metric");
  const bool frc = rule->metric == VK_METRIC_FRC_RESOLUTION;
  const bool ssim = rule->metric == VK_METRIC_SSIM_VS_PREV;
  const double spacing = rule->spacing > 0 ? rule->spacing : 1.0;
  const Geom& g = p->g;
  const int iters = rule->max_iters;
  ensure_iter_buffers(p, iters);
  p->launches = 0;
  const size_t nI = (size_t)g.Iz * g.Iy * g.Ix;
  const size_t nP = (size_t)g.Pz * g.Py * g.Px;

  const auto ta = std::chrono::steady_clock::now();
  vk::ObsStats init{};
  init.minbits = 0x7f800000u;
  init.maxbits = 0u;
  ck(cudaMemcpyAsync(p->stats.p, &init, sizeof(init), cudaMemcpyHostToDevice, s), "stats init");
  const auto tb = std::chrono::steady_clock::now();
  ck(cudaMemsetAsync(p->acc.p, 0, (size_t)iters * 4 * sizeof(double), s), "acc");
  const int sgrid = 148 * 4;
  vk::obs_stats_kernel<<<kStatBlocks, kThreads, 0, s>>>(d_obs, nI, p->stats.p, p->part.p);
  launch_check(p, "obs_stats");
  vk::reduce_partials_kernel<<<2, 256, 0, s>>>(p->part.p, kStatBlocks, 2, &p->stats.p->sr);
  launch_check(p, "obs_stats reduce");
  const auto tc = std::chrono::steady_clock::now();
  vk::ObsStats st{};
  ck(cudaMemcpyAsync(&st, p->stats.p, sizeof(st), cudaMemcpyDeviceToHost, s), "stats D2H");
  const auto tr0 = std::chrono::steady_clock::now();
  ck(cudaStreamSynchronize(s), "stats");
  const auto tr1 = std::chrono::steady_clock::now();
  if (check_obs && st.neg) fail(VK_ERR_NEGATIVE, "NegativeInput: observed image must be nonnegative");
  if (p->psf_status) fail((vk_status)p->psf_status, p->psf_msg);
  float fmin, fmax;
  std::memcpy(&fmin, &st.minbits, 4);
  std::memcpy(&fmax, &st.maxbits, 4);
  const RefStats rs{(double)nI, st.sr, st.srr, (double)fmax - (double)fmin};
  // DegenerateReference surfaces at the first metric evaluation in the
  // reference; no estimate is returned either way.
  if (!frc && !ssim) si_psnr_from_sums(rs, 0.0, 0.0, 0.0);
  if (frc) setup_frc(p);
  if (ssim) {
    setup_ssim(p, iters);
    std::vector<unsigned> r0((size_t)(iters + 1) * 2);
    for (size_t i = 0; i < r0.size(); i += 2) {
      r0[i] = 0x7f800000u;
      r0[i + 1] = 0u;
    }
    r0[0] = st.minbits;  // row 0: the observed image (the first `previous`)
    r0[1] = st.maxbits;
    ck(cudaMemcpyAsync(p->ss_range.p, r0.data(), r0.size() * sizeof(unsigned), cudaMemcpyHostToDevice, s),
       "ssim ranges");
    ck(cudaMemsetAsync(p->ss_sum.p, 0, (size_t)iters * sizeof(double), s), "ssim sums");
    ck(cudaStreamSynchronize(s), "ssim init");  // r0 is pageable
  }

  vk::pad_kernel<<<kStatBlocks, kThreads, 0, s>>>(d_obs, p->est.p, g, p->part.p, 0, g.Pz);
  launch_check(p, "pad");
  vk::reduce_partials_kernel<<<1, 256, 0, s>>>(p->part.p, kStatBlocks, 1, &p->stats.p->sump);
  launch_check(p, "pad reduce");
  if (flat_init) {
    vk::fill_mean_kernel<<<sgrid, kThreads, 0, s>>>(p->est.p, nP, p->stats.p);
    launch_check(p, "fill_mean");
  }
  x_pass(p, s, vk::XM_FWD, p->est.p, g.Pz, g.Py, g.Px, 1.0f, nullptr, nullptr, 0, nullptr,
         p->fx ? g.cx : 0);

  // Early stop is only possible from iteration patience+1 on (fails counts
  // from iteration 2); before that no host round-trip is needed.
  const bool may_stop = rule->patience + 1 <= iters;
  int run = 0;
  bool stopped = false;
  std::vector<double> values, gwall;
  // A run that may stop early decides on the device (run_graph_loop) unless
  // per-launch profiling is on or VK_RL_NO_GRAPH=1; fixed-count runs (e.g.
  // the benchmark, patience = max_iters) launch the passes directly.
  const char* nograph = std::getenv("VK_RL_NO_GRAPH");
  const bool graph = may_stop && !p->prof && !(nograph && nograph[0] == '1');
  if (graph) {
    run_graph_loop(p, s, d_obs, rule, frc, ssim, spacing, values, gwall, run, stopped);
    vk::crop_kernel<<<sgrid, kThreads, 0, s>>>(p->est.p, d_out, g);
    launch_check(p, "crop");
  }
  ck(cudaEventRecord(p->events[0], s), "event");
  for (int it = 1; it <= iters && !graph; ++it) {
    // the last iteration writes the cropped output directly unless a metric
    // still needs the updated estimate
    const bool last = it == iters && !frc && !ssim;
    conv_yz(p, s, p->otf.p);
    x_pass(p, s, vk::XM_RATIO, nullptr, g.Pz, g.Py, g.Px, 1.f, p->est.p, d_obs, it, nullptr);
    conv_yz(p, s, p->otf_flip.p);
    x_pass(p, s, last ? vk::XM_UPDATE_LAST : vk::XM_UPDATE, nullptr, g.Pz, g.Py, g.Px, 1.f, p->est.p, d_obs,
           it, last ? d_out : nullptr);
    if (frc) values.push_back(frc_eval(p, s, spacing));  // syncs: the value is needed on the host
    if (ssim) ssim_eval(p, s, it, d_obs);
    ck(cudaEventRecord(p->events[it], s), "event");
    run = it;
    if (may_stop && it >= rule->patience + 1 && it < iters) {
      if (ssim) {
        std::vector<double> sums(it);
        ck(cudaMemcpyAsync(sums.data(), p->ss_sum.p, (size_t)it * sizeof(double), cudaMemcpyDeviceToHost, s),
           "ssim D2H");
        ck(cudaStreamSynchronize(s), "iteration");
        while ((int)values.size() < it) values.push_back(sums[values.size()] / (double)nI);
      } else if (!frc) {
        flush_sums(p, s, it);
        ck(cudaMemcpyAsync(p->h_acc, p->acc.p, (size_t)it * 4 * sizeof(double), cudaMemcpyDeviceToHost, s),
           "acc D2H");
        ck(cudaStreamSynchronize(s), "iteration");
        while ((int)values.size() < it) {
          const double* a = p->h_acc + values.size() * 4;
          values.push_back(si_psnr_from_sums(rs, a[1], a[2], a[3]));
        }
      }
      stopped = rule_fires(values, it, rule);
      if (stopped) {
        vk::crop_kernel<<<sgrid, kThreads, 0, s>>>(p->est.p, d_out, g);
        launch_check(p, "crop");
        break;
      }
    }
  }
  if ((frc || ssim) && !stopped && !graph) {  // the last iteration ran in UPDATE mode: crop now
    vk::crop_kernel<<<sgrid, kThreads, 0, s>>>(p->est.p, d_out, g);
    launch_check(p, "crop");
  }
  flush_sums(p, s, run);
  ck(cudaMemcpyAsync(p->h_acc, p->acc.p, (size_t)run * 4 * sizeof(double), cudaMemcpyDeviceToHost, s), "acc D2H");
  const auto tr2 = std::chrono::steady_clock::now();
  ck(cudaStreamSynchronize(s), "run");
  if (timing_on()) {
    const auto tr3 = std::chrono::steady_clock::now();
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    std::fprintf(stderr,
                 "run_device: stats init %.3f  stats launch %.3f  stats D2H %.3f  stats wait %.3f  enqueue %.3f  "
                 "final wait %.3f ms (%llu launches)\n",
                 ms(ta, tb), ms(tb, tc), ms(tc, tr0), ms(tr0, tr1), ms(tr1, tr2), ms(tr2, tr3),
                 (unsigned long long)p->launches);
  }
  if (graph) {
    // values, stop decision and timestamps come from the device
  } else if (ssim) {
    std::vector<double> sums(run);
    ck(cudaMemcpy(sums.data(), p->ss_sum.p, (size_t)run * sizeof(double), cudaMemcpyDeviceToHost), "ssim D2H");
    values.resize(run);
    for (int k = 0; k < run; ++k) values[k] = sums[k] / (double)nI;
  } else if (!frc) {
    values.resize(run);
    for (int k = 0; k < run; ++k) {
      const double* a = p->h_acc + (size_t)k * 4;
      values[k] = si_psnr_from_sums(rs, a[1], a[2], a[3]);
    }
  }
  // The reference checks the rule after the last iteration too
  // (deconv.cpp:409-423): a run whose rule fires exactly at max_iters is
  // "converged".  Only the reason can change here (the estimate is final).
  if (!stopped) stopped = rule_fires(values, run, rule);
  prof_collect(p);
  if (trace) {
    trace->iters_run = run;
    trace->stop_reason = stopped ? 1 : 0;
    for (int i = 0; i < 3; ++i) trace->fft_shape[i] = i < p->rank ? p->wshape[i] : 0;
    for (int k = 0; k < run && k < trace->capacity; ++k) {
      const double* a = p->h_acc + (size_t)k * 4;
      if (trace->metric)
        trace->metric[k] = (frc || ssim || graph) ? values[k] : si_psnr_from_sums(rs, a[1], a[2], a[3]);
      if (trace->log_likelihood) trace->log_likelihood[k] = a[0];
      if (trace->wall_s && graph) {
        trace->wall_s[k] = gwall[k];
      } else if (trace->wall_s) {
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, p->events[k], p->events[k + 1]), "elapsed");
        trace->wall_s[k] = ms * 1e-3;
      }
    }
  }
}

// Lanes for a batch of n independent volumes: VK_RL_LANES, else enough to
// fill the GPU when one volume's x-pass grid is short of a few waves.
int lane_count(vk_rl_plan p, int n, bool host) {
  const char* env = std::getenv("VK_RL_LANES");
  int want;
  if (env && std::atoi(env) > 0) {
    want = std::atoi(env);
  } else {
    // measured on B200 with the current kernels (profiles/r01/final/lanes_*.json):
    // C3 (64x256x256 volumes) 2/3/4 lanes = 3.58/3.36/3.33e10, C5 (2048^2
    // fields) 1/2/3/4 = 3.07/3.57/3.70/3.54e10 voxel-iters/s.  (With the
    // round's first kernels, profiles/r01/lanes.log, C3 peaked at 3 lanes.)
    // Host-buffer batches: a lane's copies leave the GPU to the others, so
    // one more lane pays (C3, 8 pageable volumes: 2/3/4 lanes = 2.89/2.64-2.76/
    // 2.74 ms per volume, profiles/r02/staging_dma.md).
    want = p->rank == 2 ? 3 : (host ? 3 : 2);
  }
  return std::max(1, std::min(want, n));
}

// Runs fn(lane_plan, volume) for volumes 0..n-1, volume i on lane i % lanes,
// each lane on its own host thread and stream; rethrows the first failure.
template <class F>
void run_lanes(vk_rl_plan p, int n, bool host, F&& fn) {
  if (n <= 0) return;
  const int nl = lane_count(p, n, host);
  while ((int)p->lanes.size() < nl - 1) {
    vk_rl_plan q = create_plan(p->device, p->rank, p->ishape, p->rank, p->kshape, p->psf_host.data(), p->pad ? 1 : 0);
    q->prof = p->prof;
    p->lanes.push_back(q);
  }
  std::vector<Fail> errs(nl);
  std::vector<int> bad(nl, 0);
  std::vector<uint64_t> cnt(nl, 0);
  auto work = [&](int li) {
    vk_rl_plan q = li == 0 ? p : p->lanes[li - 1];
    try {
      DeviceGuard dg(p->device);
      for (int i = li; i < n; i += nl) {
        fn(q, i);
        cnt[li] += q->launches;
      }
    } catch (const Fail& e) {
      errs[li] = e;
      bad[li] = 1;
    } catch (const std::exception& e) {
      errs[li] = Fail{VK_ERR_ARG, e.what()};
      bad[li] = 1;
    }
  };
  std::vector<std::thread> th;
  for (int li = 1; li < nl; ++li) th.emplace_back(work, li);
  work(0);
  for (auto& t : th) t.join();
  uint64_t launches = 0;
  for (int li = 0; li < nl; ++li) launches += cnt[li];
  p->launches = launches;  // every launch of the batch
  for (int li = 0; li < nl; ++li)
    if (bad[li]) throw errs[li];
}

// filters::fft_convolve on a conv plan (filters.cpp:174-264): R2C of the
// image, times the kernel spectrum (1/prod(W) folded in), C2R and the crop at
// the kernel centre (linear) or at 0 (circular).
void conv_device(vk_rl_plan p, const float* d_img, float* d_out, cudaStream_t s) {
  if (!p->conv) fail(VK_ERR_ARG, "plan was not created by vk_conv_plan_create");
  const Geom& g = p->g;
  p->launches = 0;
  if (p->circ) {  // periodic extension -> linear 'same' convolution -> crop at h
    const size_t en = (size_t)p->circ_e[0] * p->circ_e[1] * p->circ_e[2];
    if (p->circ_in.n < en) p->circ_in.alloc(en, "circular extension");
    if (p->circ_out.n < en) p->circ_out.alloc(en, "circular result");
    vk::wrap_extend_kernel<<<148 * 4, kThreads, 0, s>>>(d_img, g.Iz, g.Iy, g.Ix, p->circ_in.p, p->circ_e[0],
                                                         p->circ_e[1], p->circ_e[2], p->circ_h[0], p->circ_h[1],
                                                         p->circ_h[2]);
    launch_check(p, "wrap extend");
    conv_device(p->circ, p->circ_in.p, p->circ_out.p, s);
    vk::crop_block_kernel<<<148 * 4, kThreads, 0, s>>>(p->circ_out.p, p->circ_e[1], p->circ_e[2], d_out, g.Iz, g.Iy,
                                                        g.Ix, p->circ_h[0], p->circ_h[1], p->circ_h[2]);
    launch_check(p, "crop block");
    p->launches += p->circ->launches;
    return;
  }
  x_pass(p, s, vk::XM_FWD, d_img, g.Pz, g.Py, g.Px, 1.0f, nullptr, nullptr, 0, nullptr, 0);
  conv_yz(p, s, p->otf.p);
  x_pass(p, s, vk::XM_CONV_OUT, nullptr, g.Pz, g.Py, g.Px, 1.f, nullptr, nullptr, 0, d_out);
}

void step_device(vk_rl_plan p, const float* d_est, const float* d_obs, float* d_out, cudaStream_t s) {
  if (p->conv) fail(VK_ERR_ARG, "plan was created for fft_convolve");
  if (p->pad) fail(VK_ERR_ARG, "rl_step needs a plan created with pad_replicate = 0");
  const Geom& g = p->g;
  ensure_iter_buffers(p, 1);
  p->launches = 0;
  ck(cudaMemsetAsync(p->acc.p, 0, 4 * sizeof(double), s), "acc");
  x_pass(p, s, vk::XM_FWD, d_est, g.Pz, g.Py, g.Px, 1.0f, nullptr, nullptr, 0, nullptr, p->fx ? g.cx : 0);
  conv_yz(p, s, p->otf.p);
  x_pass(p, s, vk::XM_RATIO, nullptr, g.Pz, g.Py, g.Px, 1.f, nullptr, d_obs, 1, nullptr);
  conv_yz(p, s, p->otf_flip.p);
  x_pass(p, s, vk::XM_UPDATE_LAST, nullptr, g.Pz, g.Py, g.Px, 1.f, const_cast<float*>(d_est), d_obs, 1,
         d_out);
}

size_t image_count(vk_rl_plan p) { return (size_t)p->g.Iz * p->g.Iy * p->g.Ix; }

// ---- plan cache -----------------------------------------------------------
// The one-shot entry points (vk_richardson_lucy, vk_rl_step_psf,
// vk_fft_convolve) replace calls that build their transforms per call
// (deconv.cpp:332, :196-200; filters.cpp:174-264).  On the CPU that is cheap;
// on the GPU a plan is ~1.3 GB of cudaMalloc plus two OTF builds at C2.  So
// plans are kept, keyed on (device, kind, shapes, PSF values), LRU, up to
// VK_RL_PLAN_CACHE plans (default 2, 0 disables).  A plan in use by another
// thread is never shared: that caller builds its own.
struct PlanKey {
  int device, rank, pad, conv;
  uint64_t shape[VK_MAX_RANK], kshape[VK_MAX_RANK];
  std::vector<float> psf;
  std::string env;  // the VK_RL_* switches read at plan creation
  bool operator==(const PlanKey& o) const {
    return device == o.device && rank == o.rank && pad == o.pad && conv == o.conv &&
           std::equal(shape, shape + rank, o.shape) && std::equal(kshape, kshape + rank, o.kshape) && psf == o.psf &&
           env == o.env;
  }
};

// Plan-shaping environment switches (sorted "NAME=value;" list): a plan built
// under other switches is a different plan.
std::string plan_env() {
  std::vector<std::string> v;
  for (char** e = environ; e && *e; ++e)
    if (std::strncmp(*e, "VK_RL_", 6) == 0 && std::strncmp(*e, "VK_RL_PLAN_CACHE=", 17) != 0 &&
        std::strncmp(*e, "VK_RL_HOST_THREADS=", 19) != 0 && std::strncmp(*e, "VK_RL_LIB=", 10) != 0)
      v.emplace_back(*e);
  std::sort(v.begin(), v.end());
  std::string s;
  for (const auto& x : v) s += x + ";";
  return s;
}

struct PlanCache {
  std::mutex mu;
  std::list<std::pair<PlanKey, vk_rl_plan>> lru;  // front = most recent
  size_t capacity() const {
    const char* e = std::getenv("VK_RL_PLAN_CACHE");
    return e ? (size_t)std::max(0, std::atoi(e)) : 2;
  }
  static PlanCache& get() {
    static PlanCache* c = new PlanCache();  // process lifetime: plans die with the context
    return *c;
  }
};

PlanKey make_key(int device, int rank, const uint64_t* shape, const uint64_t* kshape, const float* psf, int pad,
                 int conv) {
  PlanKey k{device, rank, pad, conv, {}, {}, {}, plan_env()};
  size_t kn = 1;
  for (int i = 0; i < rank; ++i) {
    k.shape[i] = shape[i];
    k.kshape[i] = kshape[i];
    kn *= kshape[i];
  }
  k.psf.assign(psf, psf + kn);
  return k;
}

// A plan for the key: a cached idle one, else a new one (created outside the lock).
vk_rl_plan acquire_plan(const PlanKey& k, int psf_rank) {
  PlanCache& c = PlanCache::get();
  if (c.capacity() > 0) {
    std::lock_guard<std::mutex> g(c.mu);
    for (auto it = c.lru.begin(); it != c.lru.end(); ++it)
      if (!it->second->busy && it->first == k) {
        it->second->busy = true;
        c.lru.splice(c.lru.begin(), c.lru, it);
        return c.lru.front().second;
      }
  }
  vk_rl_plan p = create_plan(k.device, k.rank, k.shape, psf_rank, k.kshape, k.psf.data(), k.pad, k.conv);
  p->busy = true;
  return p;
}

void release_plan(const PlanKey& k, vk_rl_plan p) {
  PlanCache& c = PlanCache::get();
  std::vector<vk_rl_plan> drop;
  {
    std::lock_guard<std::mutex> g(c.mu);
    p->busy = false;
    if (!p->cached) {
      if (c.capacity() == 0) {
        drop.push_back(p);
      } else {
        p->cached = true;
        c.lru.emplace_front(k, p);
      }
    }
    // evict idle plans beyond capacity, least recent first
    for (auto it = c.lru.end(); c.lru.size() > c.capacity() && it != c.lru.begin();) {
      --it;
      if (!it->second->busy) {
        drop.push_back(it->second);
        it = c.lru.erase(it);
      }
    }
  }
  for (vk_rl_plan q : drop) {
    DeviceGuard dg(q->device);
    delete q;
  }
}

// Runs fn(plan) on a cached plan for the key; the plan returns to the cache.
template <class F>
void with_cached_plan(const PlanKey& k, int psf_rank, F&& fn) {
  vk_rl_plan p = acquire_plan(k, psf_rank);
  try {
    fn(p);
  } catch (...) {
    release_plan(k, p);
    throw;
  }
  release_plan(k, p);
}

// Algorithmic HBM bytes of one launch of each kernel kind: every byte of
// data the kernel must move at least once (complex64 spectra in and out, the
// observed image once, the estimate in and out).  The OTF is NOT counted
// (amortisable / regenerable, reported separately:
// otf_bytes()).
uint64_t alg_bytes(vk_rl_plan p, int kind) {
  const Geom& g = p->g;
  const uint64_t Sp = (uint64_t)g.Hx * g.Pz * g.Py, Sb = (uint64_t)g.Hx * g.Pz * g.Wy;
  const uint64_t nI = image_count(p), nP = (uint64_t)g.Pz * g.Py * g.Px;
  switch (kind) {
    case VK_KIND_X_FWD: return 4 * nP + 8 * Sp;
    case VK_KIND_X_RATIO: return 16 * Sp + 4 * nI;
    case VK_KIND_X_UPDATE: return 16 * Sp + 8 * nP + 4 * nI;
    case VK_KIND_Y_FWD: return 8 * Sp + 8 * Sb;
    case VK_KIND_Z_CONV: return 16 * Sb;
    case VK_KIND_Y_INV: return 8 * Sb + 8 * Sp;
    case VK_KIND_Y_CONV: return 16 * Sp;
    case VK_KIND_YZ_DATAFLOW: return 16 * Sp;
    case VK_KIND_YZ_CLUSTER: return 16 * Sp;
    default: return 0;
  }
}

// OTF bytes one launch of `kind` reads from memory (0 when the OTF is
// rebuilt from its 1D factors, p->ofactored).
uint64_t otf_bytes(vk_rl_plan p, int kind) {
  const Geom& g = p->g;
  if (p->ofactored) return 0;
  const uint64_t So = (uint64_t)g.Hx * g.Wz * (p->ohalf ? p->owp : g.Wy);
  switch (kind) {
    case VK_KIND_Z_CONV:
    case VK_KIND_Y_CONV:
    case VK_KIND_YZ_DATAFLOW:
    case VK_KIND_YZ_CLUSTER: return 8 * So;
    default: return 0;
  }
}

}  // namespace

extern "C" {

uint64_t vk_good_size(uint64_t n) { return good_size(n); }

int vk_debug_guard_check(void) {
  if (!guard_on()) return -1;
  cudaDeviceSynchronize();
  GuardReg& g = GuardReg::get();
  std::lock_guard<std::mutex> lk(g.mu);
  long long v = g.violations;
  for (auto& e : g.live) v += GuardReg::damaged(e.first, e.second.first, e.second.second);
  return (int)std::min<long long>(v, 1 << 30);
}

const char* vk_last_error(void) { return g_last_error.c_str(); }
int vk_abi_version(void) { return VK_RL_ABI_VERSION; }

vk_status vk_rl_plan_create(int device, int rank, const uint64_t* shape, int psf_rank, const uint64_t* psf_shape,
                            const float* psf, int pad_replicate, vk_rl_plan* out) {
  return guarded([&] {
    if (!out || !shape || !psf_shape || !psf) fail(VK_ERR_ARG, "NULL argument");
    *out = create_plan(device, rank, shape, psf_rank, psf_shape, psf, pad_replicate);
  });
}

vk_status vk_rl_plan_shapes(vk_rl_plan p, int* rank, uint64_t* image_shape, uint64_t* domain_shape,
                            uint64_t* fft_shape) {
  return guarded([&] {
    if (!p) fail(VK_ERR_ARG, "NULL plan");
    if (rank) *rank = p->rank;
    for (int i = 0; i < p->rank; ++i) {
      if (image_shape) image_shape[i] = p->ishape[i];
      if (domain_shape) domain_shape[i] = p->dshape[i];
      if (fft_shape) fft_shape[i] = p->wshape[i];
    }
  });
}

vk_status vk_rl_plan_device_bytes(vk_rl_plan p, uint64_t* bytes) {
  return guarded([&] {
    if (!p || !bytes) fail(VK_ERR_ARG, "NULL argument");
    *bytes = (p->SA.n + p->SB.n + p->otf.n + p->otf_flip.n + p->ofac.n) * sizeof(float2) +
             (p->est.n + p->obs.n + p->out.n) * sizeof(float) + p->acc.n * sizeof(double) +
             p->ring2.n * sizeof(float2) + (p->xpart.n + p->part.n) * sizeof(double) +
             (p->ss_img[0].n + p->ss_img[1].n) * sizeof(float) +
             (p->ss_f[0].n + p->ss_f[1].n + p->ss_sum.n) * sizeof(double) +
             (p->frc_even.n + p->frc_odd.n) * sizeof(float);
    if (p->frc) *bytes += (p->frc->SA.n + p->frc->SB.n + p->frc->otf.n + p->frc->otf_flip.n) * sizeof(float2);
  });
}

vk_status vk_rl_plan_launches(vk_rl_plan p, uint64_t* launches) {
  return guarded([&] {
    if (!p || !launches) fail(VK_ERR_ARG, "NULL argument");
    *launches = p->launches;
  });
}

vk_status vk_rl_plan_describe(vk_rl_plan p, char* buf, int len) {
  return guarded([&] {
    if (!p || !buf || len <= 0) fail(VK_ERR_ARG, "NULL argument");
    const Geom& g = p->g;
    auto axis = [](const char* n, const vk::FastEntry* f, int L) {
      return std::string(n) + (f ? ":fast(L=" + std::to_string(L) + ")" : ":generic");
    };
    std::string s = "W=" + std::to_string(g.Wz) + "x" + std::to_string(g.Wy) + "x" + std::to_string(g.Wx) +
                    " P=" + std::to_string(g.Pz) + "x" + std::to_string(g.Py) + "x" + std::to_string(g.Px) + " " +
                    axis("x", p->fx, p->fx ? p->fx->Lx : p->xL) + " " + axis("y", p->fy, p->fy ? p->fy->Ly : p->yL) +
                    " " + axis("z", p->fz, p->fz ? p->fz->Lz : p->zL) + " yz:";
    s += p->kxc ? "kx-chunks(" + std::to_string(p->kxc) + "x" + std::to_string(p->kxs) +
                      (p->ring_window ? ",l2persist" : "") + ")"
                : g.Wz > 1 ? "3-pass" : "y-conv";
    if (p->ztma) s += " z:tma";
    if (p->ofactored) s += " otf:factored";
    if (p->ohalf) s += " otf:half";
    if (p->ytma) s += " y:bulk";
    if (p->xtma) s += " x:tma";
    std::strncpy(buf, s.c_str(), (size_t)len - 1);
    buf[len - 1] = 0;
  });
}

vk_status vk_rl_plan_profile(vk_rl_plan p, int enable) {
  return guarded([&] {
    if (!p) fail(VK_ERR_ARG, "NULL plan");
    DeviceGuard dg(p->device);
    prof_collect(p);
    p->prof = enable != 0;
    for (auto* l : p->lanes) {
      prof_collect(l);
      l->prof = p->prof;
    }
  });
}

vk_status vk_rl_plan_otf_bytes(vk_rl_plan p, int n_kinds, uint64_t* otf_bytes_per_launch) {
  return guarded([&] {
    if (!p || !otf_bytes_per_launch) fail(VK_ERR_ARG, "NULL argument");
    for (int k = 0; k < n_kinds && k < VK_KIND_COUNT; ++k)  // as profiled, else one whole-volume launch
      otf_bytes_per_launch[k] = p->prof_last_otf[k] > 0 ? (uint64_t)(p->prof_last_otf[k] + 0.5) : otf_bytes(p, k);
  });
}

vk_status vk_rl_plan_profile_read(vk_rl_plan p, int n_kinds, double* ms_total, uint64_t* launches,
                                  uint64_t* alg_bytes_per_launch, int reset) {
  return guarded([&] {
    if (!p) fail(VK_ERR_ARG, "NULL plan");
    DeviceGuard dg(p->device);
    prof_collect(p);
    for (auto* l : p->lanes) prof_collect(l);
    for (int k = 0; k < n_kinds && k < VK_KIND_COUNT; ++k) {  // summed over the batch lanes
      double ms = p->prof_ms[k], bytes = p->prof_bytes[k], otf = p->prof_otf[k];
      uint64_t cnt = p->prof_n[k];
      for (auto* l : p->lanes) {
        ms += l->prof_ms[k];
        cnt += l->prof_n[k];
        bytes += l->prof_bytes[k];
        otf += l->prof_otf[k];
      }
      if (ms_total) ms_total[k] = ms;
      if (launches) launches[k] = cnt;
      // mean algorithmic bytes of the launches profiled (chunked passes
      // launch per chunk), else one whole-volume launch's
      if (alg_bytes_per_launch) alg_bytes_per_launch[k] = cnt ? (uint64_t)(bytes / cnt + 0.5) : alg_bytes(p, k);
      if (cnt) p->prof_last_otf[k] = otf / cnt;
    }
    if (reset)
      for (int k = 0; k < VK_KIND_COUNT; ++k) {
        p->prof_ms[k] = p->prof_bytes[k] = p->prof_otf[k] = 0;
        p->prof_n[k] = 0;
        for (auto* l : p->lanes) {
          l->prof_ms[k] = l->prof_bytes[k] = l->prof_otf[k] = 0;
          l->prof_n[k] = 0;
        }
      }
  });
}

vk_status vk_rl_plan_destroy(vk_rl_plan p) {
  return guarded([&] {
    if (!p) return;
    DeviceGuard dg(p->device);
    delete p;
  });
}

vk_status vk_rl_run_device(vk_rl_plan p, const float* d_obs, float* d_est, const vk_stop_rule* rule, int flat_init,
                           vk_trace* trace, void* stream) {
  return guarded([&] {
    if (!p || !d_obs || !d_est) fail(VK_ERR_ARG, "NULL argument");
    DeviceGuard dg(p->device);
    run_device(p, d_obs, d_est, rule, flat_init, trace, (cudaStream_t)stream, true);
  });
}

vk_status vk_rl_run(vk_rl_plan p, const float* obs, float* est, const vk_stop_rule* rule, int flat_init,
                    vk_trace* trace) {
  return guarded([&] {
    if (!p || !obs || !est) fail(VK_ERR_ARG, "NULL argument");
    check_rule(rule);
    DeviceGuard dg(p->device);
    const size_t n = image_count(p);
    const bool timing = timing_on();
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    if (p->obs.n < n) p->obs.alloc(n, "observed");
    if (p->out.n < n) p->out.alloc(n, "output");
    p->staging.h2d(p->obs.p, obs, n * sizeof(float), p->stream);
    const auto t1 = clk::now();
    // a pageable output (e.g. a fresh array) is faulted in while the GPU runs
    std::thread touch;
    if (!host_pinned(est)) touch = std::thread([=] { prefault(est, n * sizeof(float)); });
    const auto t1b = clk::now();
    try {
      run_device(p, p->obs.p, p->out.p, rule, flat_init, trace, p->stream, true);
    } catch (...) {
      if (touch.joinable()) touch.join();
      throw;
    }
    const auto t2 = clk::now();
    if (touch.joinable()) touch.join();
    const auto t3 = clk::now();
    p->staging.d2h(est, p->out.p, n * sizeof(float), p->stream);
    if (timing) {
      const auto t4 = clk::now();
      auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "vk_rl_run: h2d(enqueue+host copy) %.3f  prefault spawn %.3f  run %.3f  prefault wait %.3f  d2h %.3f ms\n",
                   ms(t0, t1), ms(t1, t1b), ms(t1b, t2), ms(t2, t3), ms(t3, t4));
    }
  });
}

vk_status vk_rl_run_batch(vk_rl_plan p, int n, const float* const* obs, float* const* est, const vk_stop_rule* rule,
                          int flat_init, vk_trace* traces) {
  return guarded([&] {
    if (!p || n < 0 || (n > 0 && (!obs || !est))) fail(VK_ERR_ARG, "NULL argument");
    check_rule(rule);
    run_lanes(p, n, true, [&](vk_rl_plan q, int i) {
      const vk_status st = vk_rl_run(q, obs[i], est[i], rule, flat_init, traces ? &traces[i] : nullptr);
      if (st != VK_OK) fail(st, "volume " + std::to_string(i) + ": " + g_last_error);
    });
  });
}

vk_status vk_rl_run_batch_device(vk_rl_plan p, int n, const float* const* d_obs, float* const* d_est,
                                 const vk_stop_rule* rule, int flat_init, vk_trace* traces, void* stream) {
  return guarded([&] {
    if (!p || n < 0 || (n > 0 && (!d_obs || !d_est))) fail(VK_ERR_ARG, "NULL argument");
    check_rule(rule);
    DeviceGuard dg(p->device);
    ck(cudaStreamSynchronize((cudaStream_t)stream), "batch inputs");  // the lanes read them
    run_lanes(p, n, false, [&](vk_rl_plan q, int i) {
      run_device(q, d_obs[i], d_est[i], rule, flat_init, traces ? &traces[i] : nullptr, q->stream, true);
    });
  });
}

vk_status vk_rl_plan_lanes(vk_rl_plan p, int* lanes) {
  return guarded([&] {
    if (!p || !lanes) fail(VK_ERR_ARG, "NULL argument");
    *lanes = 1 + (int)p->lanes.size();
  });
}

vk_status vk_rl_step_device(vk_rl_plan p, const float* d_est, const float* d_obs, float* d_out, void* stream) {
  return guarded([&] {
    if (!p || !d_est || !d_obs || !d_out) fail(VK_ERR_ARG, "NULL argument");
    DeviceGuard dg(p->device);
    step_device(p, d_est, d_obs, d_out, (cudaStream_t)stream);
  });
}

vk_status vk_rl_step(vk_rl_plan p, const float* e, const float* o, float* out) {
  return guarded([&] {
    if (!p || !e || !o || !out) fail(VK_ERR_ARG, "NULL argument");
    DeviceGuard dg(p->device);
    const size_t n = image_count(p);
    if (p->obs.n < n) p->obs.alloc(n, "observed");
    if (p->out.n < n) p->out.alloc(n, "output");
    DevBuf<float> de;
    de.alloc(n, "estimate");
    p->staging.h2d(de.p, e, n * sizeof(float), p->stream);
    p->staging.h2d(p->obs.p, o, n * sizeof(float), p->stream);
    step_device(p, de.p, p->obs.p, p->out.p, p->stream);
    p->staging.d2h(out, p->out.p, n * sizeof(float), p->stream);
  });
}

vk_status vk_richardson_lucy(int device, int rank, const uint64_t* shape, const float* obs, int psf_rank,
                             const uint64_t* psf_shape, const float* psf, const vk_stop_rule* rule, int flat_init,
                             float* est, vk_trace* trace) {
  return guarded([&] {
    check_rule(rule);  // deconv.cpp:306-309
    if (rank != psf_rank) fail(VK_ERR_SHAPE, "ShapeMismatch: psf rank must match the image rank");
    if (!shape || !obs || !psf_shape || !psf || !est) fail(VK_ERR_ARG, "NULL argument");
    if (rank < 1 || rank > VK_MAX_RANK) fail(VK_ERR_ARG, "rank must be 1, 2 or 3");
    with_cached_plan(make_key(device, rank, shape, psf_shape, psf, 1, 0), psf_rank, [&](vk_rl_plan p) {
      const vk_status st = vk_rl_run(p, obs, est, rule, flat_init, trace);
      if (st != VK_OK) fail(st, g_last_error);
    });
  });
}

vk_status vk_richardson_lucy_batch(int device, int rank, const uint64_t* shape, int n, const float* const* obs,
                                   int psf_rank, const uint64_t* psf_shape, const float* psf, const vk_stop_rule* rule,
                                   int flat_init, float* const* est, vk_trace* traces) {
  return guarded([&] {
    check_rule(rule);
    if (rank != psf_rank) fail(VK_ERR_SHAPE, "ShapeMismatch: psf rank must match the image rank");
    if (!shape || !psf_shape || !psf || n < 0 || (n > 0 && (!obs || !est))) fail(VK_ERR_ARG, "NULL argument");
    if (rank < 1 || rank > VK_MAX_RANK) fail(VK_ERR_ARG, "rank must be 1, 2 or 3");
    if (n == 0) return;
    with_cached_plan(make_key(device, rank, shape, psf_shape, psf, 1, 0), psf_rank, [&](vk_rl_plan p) {
      const vk_status st = vk_rl_run_batch(p, n, obs, est, rule, flat_init, traces);
      if (st != VK_OK) fail(st, g_last_error);
    });
  });
}

vk_status vk_rl_step_psf(int device, int rank, const uint64_t* shape, const float* e, const float* o, int psf_rank,
                         const uint64_t* psf_shape, const float* psf, float* out) {
  return guarded([&] {
    if (!shape || !e || !o || !psf_shape || !psf || !out) fail(VK_ERR_ARG, "NULL argument");
    if (rank < 1 || rank > VK_MAX_RANK) fail(VK_ERR_ARG, "rank must be 1, 2 or 3");
    if (psf_rank != rank) fail(VK_ERR_SHAPE, "ShapeMismatch: psf rank must match the image rank");
    with_cached_plan(make_key(device, rank, shape, psf_shape, psf, 0, 0), psf_rank, [&](vk_rl_plan p) {
      const vk_status st = vk_rl_step(p, e, o, out);
      if (st != VK_OK) fail(st, g_last_error);
    });
  });
}

vk_status vk_plan_cache_clear(void) {
  return guarded([&] {
    PlanCache& c = PlanCache::get();
    std::vector<vk_rl_plan> drop;
    {
      std::lock_guard<std::mutex> g(c.mu);
      for (auto it = c.lru.begin(); it != c.lru.end();) {
        if (!it->second->busy) {
          drop.push_back(it->second);
          it = c.lru.erase(it);
        } else {
          it->second->cached = false;  // freed by its user on release
          it = c.lru.erase(it);
        }
      }
    }
    for (vk_rl_plan q : drop) {
      DeviceGuard dg(q->device);
      delete q;
    }
  });
}

// ---- single-volume slab decomposition ---------------------
// The P domain is cut into z slabs; slab r owns P rows [z0, z1) and computes
// on Q = [z0 - hb, z1 + ha) clipped to [0, Pz), hb = Kz-1-cz, ha = cz (the
// reach of both correlations, deconv.cpp:40,126-130).  The convolution over Q
// with zeros outside equals the full one on the owned rows once the halo rows
// hold the neighbours' values; both exchanges (estimate before the forward
// correlation, ratio before the backward one) happen in the x-transformed
// spectrum S_A right after an x pass, because the x transform acts on each
// (z, y) row alone.  The plan's image is the slab's own image rows.

void slab_geometry(const uint64_t* shape3, const uint64_t* kshape3, int nslabs, int r, int* out) {
  const int Kz = (int)kshape3[0], Iz = (int)shape3[0];
  const int ozg = Kz / 2, Pz = Iz + 2 * ozg, cz = (Kz - 1) / 2;
  const int hb = Kz - 1 - cz, ha = cz;
  if (nslabs < 1 || r < 0 || r >= nslabs) fail(VK_ERR_ARG, "bad slab index");
  const int z0 = (int)((long long)Pz * r / nslabs), z1 = (int)((long long)Pz * (r + 1) / nslabs);
  const int q0 = std::max(0, z0 - hb), q1 = std::min(Pz, z1 + ha);
  // own image rows (P row z <-> I row z - ozg)
  const int i0 = std::max(0, z0 - ozg), i1 = std::min(Iz, z1 - ozg);
  if (z1 - z0 < std::max(hb, ha) || i1 <= i0)
    fail(VK_ERR_ARG, "too many slabs: each slab needs >= max(halo) P rows and one image row");
  out[0] = z0;       // own P rows, global
  out[1] = z1;
  out[2] = q0;       // local domain, global P rows
  out[3] = q1;
  out[4] = i0;       // own image rows
  out[5] = i1;
}

vk_status vk_conv_plan_create(int device, int rank, const uint64_t* shape, int kernel_rank,
                              const uint64_t* kernel_shape, const float* kernel, int circular, vk_rl_plan* out) {
  return guarded([&] {
    if (!shape || !kernel_shape || !kernel || !out) fail(VK_ERR_ARG, "NULL argument");
    *out = create_plan(device, rank, shape, kernel_rank, kernel_shape, kernel, 0, circular ? 2 : 1);
  });
}

vk_status vk_conv_run_device(vk_rl_plan p, const float* d_img, float* d_out, void* stream) {
  return guarded([&] {
    if (!p || !d_img || !d_out) fail(VK_ERR_ARG, "NULL argument");
    DeviceGuard dg(p->device);
    conv_device(p, d_img, d_out, (cudaStream_t)stream);
  });
}

vk_status vk_conv_run(vk_rl_plan p, const float* img, float* out) {
  return guarded([&] {
    if (!p || !img || !out) fail(VK_ERR_ARG, "NULL argument");
    DeviceGuard dg(p->device);
    const size_t n = image_count(p);
    if (p->obs.n < n) p->obs.alloc(n, "image");
    if (p->out.n < n) p->out.alloc(n, "output");
    p->staging.h2d(p->obs.p, img, n * sizeof(float), p->stream);
    conv_device(p, p->obs.p, p->out.p, p->stream);
    p->staging.d2h(out, p->out.p, n * sizeof(float), p->stream);
  });
}

vk_status vk_fft_convolve(int device, int rank, const uint64_t* shape, const float* img, int kernel_rank,
                          const uint64_t* kernel_shape, const float* kernel, int circular, float* out) {
  return guarded([&] {
    if (!shape || !kernel_shape || !kernel || !img || !out) fail(VK_ERR_ARG, "NULL argument");
    if (rank < 1 || rank > VK_MAX_RANK) fail(VK_ERR_ARG, "rank must be 1, 2 or 3");
    if (kernel_rank != rank) fail(VK_ERR_SHAPE, "ShapeMismatch: fft_convolve: rank mismatch");
    with_cached_plan(make_key(device, rank, shape, kernel_shape, kernel, 0, circular ? 2 : 1), kernel_rank,
                     [&](vk_rl_plan p) {
                       const vk_status st = vk_conv_run(p, img, out);
                       if (st != VK_OK) fail(st, g_last_error);
                     });
  });
}

vk_status vk_rl_slab_plan_create(int device, const uint64_t* shape, const uint64_t* psf_shape, const float* psf,
                                 int nslabs, int slab, vk_rl_plan* out, vk_slab_info* info) {
  return guarded([&] {
    if (!shape || !psf_shape || !psf || !out) fail(VK_ERR_ARG, "NULL argument");
    int gm[6];
    slab_geometry(shape, psf_shape, nslabs, slab, gm);
    const uint64_t local[3] = {(uint64_t)(gm[5] - gm[4]), shape[1], shape[2]};
    const int ozg = (int)psf_shape[0] / 2;
    const int zs[2] = {gm[3] - gm[2], gm[4] + ozg - gm[2]};
    vk_rl_plan p = create_plan(device, 3, local, 3, psf_shape, psf, 1, 0, zs);
    p->slab = true;
    p->own0 = gm[0] - gm[2];
    p->own1 = gm[1] - gm[2];
    *out = p;
    if (info) {
      info->own_begin = gm[0];
      info->own_end = gm[1];
      info->domain_begin = gm[2];
      info->domain_end = gm[3];
      info->image_begin = gm[4];
      info->image_end = gm[5];
      info->halo_below = p->own0;
      info->halo_above = (gm[3] - gm[2]) - p->own1;
      info->spectrum = p->SA.p;
      info->kx_planes = (uint64_t)p->g.Hx;
      info->rows = (uint64_t)p->g.Pz;
      info->row_elems = (uint64_t)p->g.Py;
    }
  });
}

vk_status vk_rl_slab_begin(vk_rl_plan p, const float* d_obs, double* stats, void* stream) {
  return guarded([&] {
    if (!p || !p->slab || !d_obs || !stats) fail(VK_ERR_ARG, "not a slab plan / NULL argument");
    DeviceGuard dg(p->device);
    cudaStream_t s = (cudaStream_t)stream;
    const Geom& g = p->g;
    const size_t nI = (size_t)g.Iz * g.Iy * g.Ix;
    p->launches = 0;
    vk::ObsStats init{};
    init.minbits = 0x7f800000u;
    init.maxbits = 0u;
    ck(cudaMemcpyAsync(p->stats.p, &init, sizeof(init), cudaMemcpyHostToDevice, s), "stats init");
    if (!p->part.p) p->part.alloc((size_t)kStatBlocks * 8, "block partials");
    vk::obs_stats_kernel<<<kStatBlocks, kThreads, 0, s>>>(d_obs, nI, p->stats.p, p->part.p);
    launch_check(p, "obs_stats");
    vk::reduce_partials_kernel<<<2, 256, 0, s>>>(p->part.p, kStatBlocks, 2, &p->stats.p->sr);
    launch_check(p, "obs_stats reduce");
    vk::pad_kernel<<<kStatBlocks, kThreads, 0, s>>>(d_obs, p->est.p, g, p->part.p, p->own0, p->own1);
    launch_check(p, "pad");
    vk::reduce_partials_kernel<<<1, 256, 0, s>>>(p->part.p, kStatBlocks, 1, &p->stats.p->sump);
    launch_check(p, "pad reduce");
    vk::ObsStats st{};
    ck(cudaMemcpyAsync(&st, p->stats.p, sizeof(st), cudaMemcpyDeviceToHost, s), "stats D2H");
    ck(cudaStreamSynchronize(s), "stats");
    float fmin, fmax;
    std::memcpy(&fmin, &st.minbits, 4);
    std::memcpy(&fmax, &st.maxbits, 4);
    stats[0] = st.sr;
    stats[1] = st.srr;
    stats[2] = fmin;
    stats[3] = fmax;
    stats[4] = st.sump;
    stats[5] = st.neg ? 1.0 : 0.0;
    stats[6] = (double)nI;
    stats[7] = (double)(p->own1 - p->own0) * g.Py * g.Px;
  });
}

vk_status vk_rl_slab_start(vk_rl_plan p, int iters, int flat_init, double mean, void* stream) {
  return guarded([&] {
    if (!p || !p->slab) fail(VK_ERR_ARG, "not a slab plan");
    DeviceGuard dg(p->device);
    cudaStream_t s = (cudaStream_t)stream;
    const Geom& g = p->g;
    ensure_iter_buffers(p, iters);
    ck(cudaMemsetAsync(p->acc.p, 0, (size_t)iters * 4 * sizeof(double), s), "acc");
    if (flat_init) {  // mean of the whole padded volume, evaluated in double then f32 (deconv.cpp:337-341)
      vk::fill_value_kernel<<<148 * 4, kThreads, 0, s>>>(p->est.p, (size_t)g.Pz * g.Py * g.Px, (float)mean);
      launch_check(p, "fill");
    }
    x_pass(p, s, vk::XM_FWD, p->est.p, g.Pz, g.Py, g.Px, 1.0f, nullptr, nullptr, 0, nullptr,
           p->fx ? g.cx : 0);
  });
}

vk_status vk_rl_slab_forward(vk_rl_plan p, const float* d_obs, int it, void* stream) {
  return guarded([&] {
    if (!p || !p->slab || !d_obs || it < 1 || it > p->acc_cap) fail(VK_ERR_ARG, "bad slab call");
    DeviceGuard dg(p->device);
    cudaStream_t s = (cudaStream_t)stream;
    const Geom& g = p->g;
    conv_yz(p, s, p->otf.p);
    x_pass(p, s, vk::XM_RATIO, nullptr, g.Pz, g.Py, g.Px, 1.f, p->est.p, d_obs, it, nullptr);
  });
}

vk_status vk_rl_slab_backward(vk_rl_plan p, const float* d_obs, int it, float* d_out, void* stream) {
  return guarded([&] {
    if (!p || !p->slab || !d_obs || it < 1 || it > p->acc_cap) fail(VK_ERR_ARG, "bad slab call");
    DeviceGuard dg(p->device);
    cudaStream_t s = (cudaStream_t)stream;
    const Geom& g = p->g;
    conv_yz(p, s, p->otf_flip.p);
    x_pass(p, s, d_out ? vk::XM_UPDATE_LAST : vk::XM_UPDATE, nullptr, g.Pz, g.Py, g.Px, 1.f, p->est.p, d_obs,
           it, d_out);
  });
}

vk_status vk_rl_slab_crop(vk_rl_plan p, float* d_out, void* stream) {
  return guarded([&] {
    if (!p || !p->slab || !d_out) fail(VK_ERR_ARG, "bad slab call");
    DeviceGuard dg(p->device);
    vk::crop_kernel<<<148 * 4, kThreads, 0, (cudaStream_t)stream>>>(p->est.p, d_out, p->g);
    launch_check(p, "crop");
  });
}

// S_A rows [row, row + n) of every kx plane <-> a packed [Hx][n][Py] buffer,
// or straight into another slab plan's rows (same device or a peer, UVA).
void slab_rows_check(vk_rl_plan p, int row, int n) {
  if (!p || !p->slab) fail(VK_ERR_ARG, "not a slab plan");
  if (row < 0 || n < 0 || row + n > p->g.Pz) fail(VK_ERR_ARG, "slab rows out of range");
}

vk_status vk_rl_slab_pack(vk_rl_plan p, int row, int n, void* d_buf, void* stream) {
  return guarded([&] {
    slab_rows_check(p, row, n);
    if (n == 0) return;
    DeviceGuard dg(p->device);
    const size_t w = (size_t)n * p->g.Py * sizeof(float2), pitch = (size_t)p->g.Pz * p->g.Py * sizeof(float2);
    ck(cudaMemcpy2DAsync(d_buf, w, p->SA.p + (size_t)row * p->g.Py, pitch, w, p->g.Hx, cudaMemcpyDeviceToDevice,
                         (cudaStream_t)stream),
       "slab pack");
  });
}

vk_status vk_rl_slab_unpack(vk_rl_plan p, int row, int n, const void* d_buf, void* stream) {
  return guarded([&] {
    slab_rows_check(p, row, n);
    if (n == 0) return;
    DeviceGuard dg(p->device);
    const size_t w = (size_t)n * p->g.Py * sizeof(float2), pitch = (size_t)p->g.Pz * p->g.Py * sizeof(float2);
    ck(cudaMemcpy2DAsync(p->SA.p + (size_t)row * p->g.Py, pitch, d_buf, w, w, p->g.Hx, cudaMemcpyDeviceToDevice,
                         (cudaStream_t)stream),
       "slab unpack");
  });
}

vk_status vk_rl_slab_copy_rows(vk_rl_plan src, int src_row, vk_rl_plan dst, int dst_row, int n, void* stream) {
  return guarded([&] {
    slab_rows_check(src, src_row, n);
    slab_rows_check(dst, dst_row, n);
    if (src->g.Hx != dst->g.Hx || src->g.Py != dst->g.Py) fail(VK_ERR_SHAPE, "ShapeMismatch: slab planes differ");
    if (n == 0) return;
    DeviceGuard dg(dst->device);
    const size_t w = (size_t)n * src->g.Py * sizeof(float2);
    ck(cudaMemcpy2DAsync(dst->SA.p + (size_t)dst_row * dst->g.Py, (size_t)dst->g.Pz * dst->g.Py * sizeof(float2),
                         src->SA.p + (size_t)src_row * src->g.Py, (size_t)src->g.Pz * src->g.Py * sizeof(float2), w,
                         src->g.Hx, cudaMemcpyDefault, (cudaStream_t)stream),
       "slab copy");
  });
}

vk_status vk_rl_slab_sums(vk_rl_plan p, int iters, double* acc, void* stream) {
  return guarded([&] {
    if (!p || !p->slab || !acc || iters < 0 || iters > p->acc_cap) fail(VK_ERR_ARG, "bad slab call");
    DeviceGuard dg(p->device);
    flush_sums(p, (cudaStream_t)stream, iters);
    ck(cudaMemcpyAsync(acc, p->acc.p, (size_t)iters * 4 * sizeof(double), cudaMemcpyDeviceToHost,
                       (cudaStream_t)stream),
       "acc D2H");
    ck(cudaStreamSynchronize((cudaStream_t)stream), "acc");
  });
}

}  // extern "C"

// stager.cu — pipelined host→device staging for the drop-in boundary.
//
// The reference's relations are ordinary (pageable) numpy columns. A plain
// cudaMemcpy from pageable memory runs at ~11 GB/s on the B200 box, while a
// copy from pinned memory reaches ~55 GB/s and 8 host threads copy memory at
// ~50 GB/s. The stager overlaps the two: a pool of native threads copies
// chunk c of the source into a pinned ring slot while the copy engine DMAs
// chunk c-1 to HBM on the stager's own copy stream. The caller's compute
// stream is made to wait (cudaStreamWaitEvent) for the finished upload, so
// kernels that consume the column are ordered after it while unrelated
// kernels already queued keep running — uploading the payload columns
// overlaps the key sort.
#include <algorithm>
#include <cerrno>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

#include "common.cuh"

namespace rl {
namespace stage {

class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return int(workers_.size()); }
  // run fn(i) for i in [0, size()) on the workers; returns when all finished.
  // Callers from several host threads take turns (job_/pending_/gen_ belong to
  // one job at a time; ctypes releases the GIL, so two calls can overlap).
  void parallel(const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> one_job(job_mu_);
    std::unique_lock<std::mutex> lk(m_);
    job_ = &fn;
    pending_ = int(workers_.size());
    ++gen_;
    cv_.notify_all();
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int idx) {
    uint64_t seen = 0;
    while (true) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
      }
      if (job) (*job)(idx);
      {
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex job_mu_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

struct Stager {
  Pool pool;
  size_t chunk;
  int slots;
  char* ring = nullptr;
  std::vector<cudaEvent_t> slot_free;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t done = nullptr;
  int next_slot = 0;
  std::mutex call_mu;  // one upload at a time per stager

  Stager(int threads, size_t chunk_bytes, int n_slots) : pool(threads), chunk(chunk_bytes), slots(n_slots) {}
};

}  // namespace stage
}  // namespace rl

using rl::stage::Stager;

extern "C" {

RL_API void* rl_stager_create(int32_t threads, size_t chunk_bytes, int32_t slots) {
  if (threads < 1 || slots < 2 || chunk_bytes < 4096) return nullptr;
  Stager* s = new Stager(threads, chunk_bytes, slots);
  bool ok = cudaHostAlloc(reinterpret_cast<void**>(&s->ring), chunk_bytes * size_t(slots), cudaHostAllocDefault) ==
                cudaSuccess &&
            cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming) == cudaSuccess;
  s->slot_free.resize(slots);
  for (int i = 0; ok && i < slots; ++i)
    ok = cudaEventCreateWithFlags(&s->slot_free[i], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    delete s;
    return nullptr;
  }
  for (int i = 0; i < slots; ++i) cudaEventRecord(s->slot_free[i], s->copy_stream);
  return s;
}

RL_API void rl_stager_destroy(void* handle) {
  Stager* s = static_cast<Stager*>(handle);
  if (!s) return;
  if (s->copy_stream) cudaStreamSynchronize(s->copy_stream);
  for (auto e : s->slot_free)
    if (e) cudaEventDestroy(e);
  if (s->done) cudaEventDestroy(s->done);
  if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
  if (s->ring) cudaFreeHost(s->ring);
  delete s;
}

// Page-lock a long-lived host buffer so uploads from it are one direct DMA
// (no staging copy: the staging memcpy + DMA triple the host memory traffic).
RL_API int rl_host_register(void* host, size_t bytes) {
  if (!host || !bytes) return RL_ERR_BAD_ARG;
  cudaError_t e = cudaHostRegister(host, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) cudaGetLastError();
  return rl::rl_cuda_status(e);
}

// 1 if `host` lies in page-locked memory this process registered or
// allocated pinned (e.g. a previous operator's output), else 0.
RL_API int rl_host_is_pinned(const void* host) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, host) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return attr.type == cudaMemoryTypeHost ? 1 : 0;
}

RL_API int rl_host_unregister(void* host) {
  cudaError_t e = cudaHostUnregister(host);
  if (e != cudaSuccess) cudaGetLastError();
  return rl::rl_cuda_status(e);
}

// Upload from page-locked (registered or pinned) memory: one DMA on the
// stager's copy stream, ordered like rl_stager_h2d.
RL_API int rl_stager_h2d_pinned(void* handle, void* dst_dev, const void* src_host, size_t bytes, void* stream,
                                void* ready_event) {
  Stager* s = static_cast<Stager*>(handle);
  if (!s || (bytes && (!dst_dev || !src_host))) return RL_ERR_BAD_ARG;
  if (bytes == 0) return RL_OK;
  std::lock_guard<std::mutex> g(s->call_mu);
  cudaError_t e = cudaSuccess;
  if (ready_event) e = cudaStreamWaitEvent(s->copy_stream, static_cast<cudaEvent_t>(ready_event), 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, s->copy_stream);
  if (e == cudaSuccess) e = cudaEventRecord(s->done, s->copy_stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), s->done, 0);
  return rl::rl_cuda_status(e);
}

// Wait until every upload issued so far has finished reading host memory.
RL_API int rl_stager_drain(void* handle) {
  Stager* s = static_cast<Stager*>(handle);
  if (!s) return RL_ERR_BAD_ARG;
  return rl::rl_cuda_status(cudaStreamSynchronize(s->copy_stream));
}

RL_API int rl_stager_h2d(void* handle, void* dst_dev, const void* src_host, size_t bytes, void* stream,
                         void* ready_event) {
  Stager* s = static_cast<Stager*>(handle);
  if (!s || (bytes && (!dst_dev || !src_host))) return RL_ERR_BAD_ARG;
  if (bytes == 0) return RL_OK;
  std::lock_guard<std::mutex> g(s->call_mu);
  if (ready_event) {  // dst may have been freed by work queued before the event: wait for it
    cudaError_t e = cudaStreamWaitEvent(s->copy_stream, static_cast<cudaEvent_t>(ready_event), 0);
    if (e != cudaSuccess) return rl::rl_cuda_status(e);
  }
  const int nt = s->pool.size();
  for (size_t off = 0; off < bytes; off += s->chunk) {
    const size_t len = std::min(s->chunk, bytes - off);
    const int slot = s->next_slot;
    s->next_slot = (s->next_slot + 1) % s->slots;
    cudaError_t e = cudaEventSynchronize(s->slot_free[slot]);  // its previous DMA has drained
    if (e != cudaSuccess) return rl::rl_cuda_status(e);
    char* dst = s->ring + size_t(slot) * s->chunk;
    const char* src = static_cast<const char*>(src_host) + off;
    if (len >= (size_t(1) << 20) && nt > 1) {
      const size_t piece = (len + nt - 1) / nt;
      s->pool.parallel([&](int i) {
        const size_t a = std::min(len, size_t(i) * piece), b = std::min(len, a + piece);
        if (b > a) std::memcpy(dst + a, src + a, b - a);
      });
    } else {
      std::memcpy(dst, src, len);
    }
    e = cudaMemcpyAsync(static_cast<char*>(dst_dev) + off, dst, len, cudaMemcpyHostToDevice, s->copy_stream);
    if (e != cudaSuccess) return rl::rl_cuda_status(e);
    cudaEventRecord(s->slot_free[slot], s->copy_stream);
  }
  cudaEventRecord(s->done, s->copy_stream);
  return rl::rl_cuda_status(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), s->done, 0));
}

// ---- RELCOL01 relation files straight to / from HBM (relation.py:364-419):
// a column section of `bytes` at `file_offset` of the open file `fd` is read
// by the pool threads with pread() into the pinned ring — each chunk split
// across the threads — while the copy engine DMAs the previous chunk; no
// numpy array, no pageable intermediate. The write direction DMAs a chunk
// into the ring and the threads pwrite() it.
static bool pread_all(int fd, char* dst, size_t len, uint64_t off) {
  while (len) {
    const ssize_t r = pread(fd, dst, len, off_t(off));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    dst += r;
    off += uint64_t(r);
    len -= size_t(r);
  }
  return true;
}

static bool pwrite_all(int fd, const char* src, size_t len, uint64_t off) {
  while (len) {
    const ssize_t r = pwrite(fd, src, len, off_t(off));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    src += r;
    off += uint64_t(r);
    len -= size_t(r);
  }
  return true;
}

RL_API int rl_stager_file_h2d(void* handle, void* dst_dev, int32_t fd, uint64_t file_offset, size_t bytes,
                              void* stream, void* ready_event) {
  Stager* s = static_cast<Stager*>(handle);
  if (!s || fd < 0 || (bytes && !dst_dev)) return RL_ERR_BAD_ARG;
  if (bytes == 0) return RL_OK;
  std::lock_guard<std::mutex> g(s->call_mu);
  if (ready_event) {
    cudaError_t e = cudaStreamWaitEvent(s->copy_stream, static_cast<cudaEvent_t>(ready_event), 0);
    if (e != cudaSuccess) return rl::rl_cuda_status(e);
  }
  const int nt = s->pool.size();
  for (size_t off = 0; off < bytes; off += s->chunk) {
    const size_t len = std::min(s->chunk, bytes - off);
    const int slot = s->next_slot;
    s->next_slot = (s->next_slot + 1) % s->slots;
    cudaError_t e = cudaEventSynchronize(s->slot_free[slot]);
    if (e != cudaSuccess) return rl::rl_cuda_status(e);
    char* dst = s->ring + size_t(slot) * s->chunk;
    bool ok = true;
    std::mutex ok_mu;
    const size_t piece = (len + nt - 1) / nt;
    s->pool.parallel([&](int i) {
      const size_t a = std::min(len, size_t(i) * piece), b = std::min(len, a + piece);
      if (b > a && !pread_all(fd, dst + a, b - a, file_offset + off + a)) {
        std::lock_guard<std::mutex> lk(ok_mu);
        ok = false;
      }
    });
    if (!ok) return RL_ERR_IO;
    e = cudaMemcpyAsync(static_cast<char*>(dst_dev) + off, dst, len, cudaMemcpyHostToDevice, s->copy_stream);
    if (e != cudaSuccess) return rl::rl_cuda_status(e);
    cudaEventRecord(s->slot_free[slot], s->copy_stream);
  }
  cudaEventRecord(s->done, s->copy_stream);
  return rl::rl_cuda_status(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), s->done, 0));
}

// File section -> host memory (e.g. page-locked columns), the threads
// splitting the section between them.
RL_API int rl_stager_file_read(void* handle, void* dst_host, int32_t fd, uint64_t file_offset, size_t bytes) {
  Stager* s = static_cast<Stager*>(handle);
  if (!s || fd < 0 || (bytes && !dst_host)) return RL_ERR_BAD_ARG;
  if (bytes == 0) return RL_OK;
  const int nt = s->pool.size();
  bool ok = true;
  std::mutex ok_mu;
  const size_t piece = (bytes + nt - 1) / nt;
  s->pool.parallel([&](int i) {
    const size_t a = std::min(bytes, size_t(i) * piece), b = std::min(bytes, a + piece);
    if (b > a && !pread_all(fd, static_cast<char*>(dst_host) + a, b - a, file_offset + a)) {
      std::lock_guard<std::mutex> lk(ok_mu);
      ok = false;
    }
  });
  return ok ? RL_OK : RL_ERR_IO;
}

// Device column -> file section. Synchronous (returns after the data is in
// the file): the DMA of chunk c+1 overlaps the pwrite of chunk c.
RL_API int rl_stager_file_d2h(void* handle, const void* src_dev, int32_t fd, uint64_t file_offset, size_t bytes,
                              void* stream) {
  Stager* s = static_cast<Stager*>(handle);
  if (!s || fd < 0 || (bytes && !src_dev)) return RL_ERR_BAD_ARG;
  if (bytes == 0) return RL_OK;
  std::lock_guard<std::mutex> g(s->call_mu);
  cudaError_t e = cudaEventRecord(s->done, static_cast<cudaStream_t>(stream));  // producers of src_dev first
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s->copy_stream, s->done, 0);
  if (e != cudaSuccess) return rl::rl_cuda_status(e);
  const int nt = s->pool.size();
  const size_t nchunks = (bytes + s->chunk - 1) / s->chunk;
  std::vector<int> slot_of(nchunks);
  auto issue = [&](size_t c) -> cudaError_t {
    const size_t off = c * s->chunk, len = std::min(s->chunk, bytes - off);
    const int slot = s->next_slot;
    s->next_slot = (s->next_slot + 1) % s->slots;
    slot_of[c] = slot;
    cudaError_t err = cudaEventSynchronize(s->slot_free[slot]);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(s->ring + size_t(slot) * s->chunk, static_cast<const char*>(src_dev) + off, len,
                            cudaMemcpyDeviceToHost, s->copy_stream);
    if (err == cudaSuccess) err = cudaEventRecord(s->slot_free[slot], s->copy_stream);
    return err;
  };
  if (nchunks) e = issue(0);
  for (size_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
    if (c + 1 < nchunks && s->slots > 1) e = issue(c + 1);  // next DMA in flight while this chunk is written
    if (e != cudaSuccess) break;
    const int slot = slot_of[c];
    e = cudaEventSynchronize(s->slot_free[slot]);
    if (e != cudaSuccess) break;
    const size_t off = c * s->chunk, len = std::min(s->chunk, bytes - off);
    const char* src = s->ring + size_t(slot) * s->chunk;
    bool ok = true;
    std::mutex ok_mu;
    const size_t piece = (len + nt - 1) / nt;
    s->pool.parallel([&](int i) {
      const size_t a = std::min(len, size_t(i) * piece), b = std::min(len, a + piece);
      if (b > a && !pwrite_all(fd, src + a, b - a, file_offset + off + a)) {
        std::lock_guard<std::mutex> lk(ok_mu);
        ok = false;
      }
    });
    if (!ok) return RL_ERR_IO;
  }
  return rl::rl_cuda_status(e);
}

}  // extern "C"

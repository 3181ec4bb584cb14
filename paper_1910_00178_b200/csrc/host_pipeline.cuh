// host_pipeline.cuh — GEMMs on HOST buffers (the reference-facing entries: gemm_conventional on
// MatrixBufs, gemm_ngemm with a resident weight, the C-ABI *_host calls), pipelined so that the
// PCIe copies in both directions and the tensor-core work overlap.
//
// C is computed in a grid of tiles (column passes j over row blocks i).  A's row blocks and B's
// row blocks (= C's column blocks) stream in on a copy-in stream in first-use order; each tile's
// GEMM runs on a compute stream once its operands have landed; its C tile leaves on a copy-out
// stream.  PCIe is full duplex, so the call approaches max(H2D, D2H) + the first tile's inputs:
//   * streamed A: the first column block is >= K/4 wide, so pass 0 produces C at least as fast as
//     A arrives (4·w0 bytes of C per K bytes of A) and the copy-out never starves; the row blocks
//     grow 256, 512, 1024, ... so the first C bytes leave after ~w0·K + 256·K input bytes;
//   * resident A (the packed weight of gemm_ngemm stays in HBM): only B streams; the first column
//     block is narrow (1024) so the copy-out starts after 1024·K bytes.
// Pageable host memory (std::vector-backed MatrixBufs) cannot be DMA'd directly: it moves through
// a ring of pinned staging slots, filled / drained by a small pool of host threads (parallel
// memcpy) — the input side on the calling thread, the output side on a second thread that
// drains C tiles as soon as their D2H into a slot completes.  Pinned operands are copied
// directly.  Every copy is stream-ordered; nothing runs on the legacy default stream.
#pragma once

#include <condition_variable>
#include <deque>
#include <functional>

#include <immintrin.h>

namespace {

// ---------------------------------------------------------------- host copy workers
// Persistent host threads for parallel memcpy (pageable <-> pinned staging).  run() splits a job
// into parts, queues them, and the caller helps until its parts are done, so concurrent callers
// (the input and output sides of one call, or several calls) never deadlock.
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool* p = new CopyPool();  // never destroyed: workers may outlive static dtors
        return *p;
    }
    int width() const { return nthreads_ + 1; }
    void run(int parts, const std::function<void(int)>& fn) {
        if (parts <= 1) {
            if (parts == 1) fn(0);
            return;
        }
        struct Job {
            std::atomic<int> left;
        };
        auto job = std::make_shared<Job>();
        job->left.store(parts);
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (int p = 1; p < parts; ++p)
                q_.push_back([job, &fn, p] {
                    fn(p);
                    job->left.fetch_sub(1);
                });
        }
        cv_.notify_all();
        fn(0);
        job->left.fetch_sub(1);
        while (job->left.load() > 0) {  // help with queued parts (ours or another caller's)
            std::function<void()> t;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (!q_.empty()) {
                    t = std::move(q_.front());
                    q_.pop_front();
                }
            }
            if (t) t();
            else std::this_thread::yield();
        }
    }

private:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        // measured on the 16-thread GPU host (profiles/r2/e2e_probe.log): 12 copying threads (11
        // workers + the caller) with 8 staging slots per direction beat 8 and 16
        nthreads_ = static_cast<int>(std::max(2u, std::min(15u, hw >= 4 ? hw * 3 / 4 - 1 : 2u)));
        if (const char* e = std::getenv("NGEMM_COPY_THREADS")) nthreads_ = std::max(1, std::atoi(e));  // experiments
        for (int i = 0; i < nthreads_; ++i)
            std::thread([this] {
                for (;;) {
                    std::function<void()> t;
                    {
                        std::unique_lock<std::mutex> lk(mu_);
                        cv_.wait(lk, [this] { return !q_.empty(); });
                        t = std::move(q_.front());
                        q_.pop_front();
                    }
                    t();
                }
            }).detach();
    }
    int nthreads_ = 2;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
};

// Large copies with non-temporal (streaming) stores: the destination is not read back by this
// thread, so skipping the read-for-ownership saves a third of the host DRAM traffic.
__attribute__((target("avx2"))) void stream_copy_avx2(uint8_t* dst, const uint8_t* src, size_t bytes) {
    const size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
    if (head >= bytes) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    bytes -= head;
    size_t i = 0;
    for (; i + 128 <= bytes; i += 128) {
        const __m256i v0 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        const __m256i v1 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
        const __m256i v2 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
        const __m256i v3 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), v0);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), v1);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), v2);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), v3);
    }
    std::memcpy(dst + i, src + i, bytes - i);
    _mm_sfence();
}

void big_copy(void* dst, const void* src, size_t bytes) {
    static const bool avx2 = __builtin_cpu_supports("avx2") && !std::getenv("NGEMM_COPY_PLAIN");
    if (avx2 && bytes >= 4096) stream_copy_avx2(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes);
    else std::memcpy(dst, src, bytes);
}

// rows x width bytes from (src, spitch) to (dst, dpitch), split over the copy pool
void par_copy_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t rows) {
    CopyPool& pool = CopyPool::get();
    const int64_t bytes = width * rows;
    const int parts = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(pool.width(), bytes >> 20)));
    pool.run(parts, [&](int p) {
        const int64_t r0 = rows * p / parts, r1 = rows * (p + 1) / parts;
        if (dpitch == width && spitch == width) {
            big_copy(static_cast<uint8_t*>(dst) + r0 * width, static_cast<const uint8_t*>(src) + r0 * width,
                     static_cast<size_t>((r1 - r0) * width));
            return;
        }
        for (int64_t r = r0; r < r1; ++r)
            big_copy(static_cast<uint8_t*>(dst) + r * dpitch, static_cast<const uint8_t*>(src) + r * spitch,
                     static_cast<size_t>(width));
    });
}

// ---------------------------------------------------------------- pinned staging slots
// Process-wide cache of pinned staging buffers (cudaHostAlloc is slow: slots are reused).
constexpr size_t kSlotBytes = 8u << 20;
struct Slot {
    uint8_t* p = nullptr;
    cudaEvent_t ev = nullptr;  // last DMA that used this slot (an event of device `dev`)
    int dev = -1;
};
std::mutex g_slot_mu;
std::vector<Slot> g_slots;

bool take_slots(int count, std::vector<Slot>& out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_slot_mu);
    while (static_cast<int>(out.size()) < count) {
        Slot s;
        auto it = std::find_if(g_slots.begin(), g_slots.end(), [dev](const Slot& x) { return x.dev == dev; });
        if (it != g_slots.end()) {
            s = *it;
            g_slots.erase(it);
        } else {
            s.dev = dev;
            if (cudaHostAlloc(reinterpret_cast<void**>(&s.p), kSlotBytes, cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            if (cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming | cudaEventBlockingSync) != cudaSuccess) {
                cudaFreeHost(s.p);
                cudaGetLastError();
                return false;
            }
        }
        out.push_back(s);
    }
    return true;
}
void give_slots(std::vector<Slot>& s) {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    for (auto& x : s) g_slots.push_back(x);
    s.clear();
}

// rows x cols int32 block (row pitch n on both sides) from this device to `dst` on device dst_dev:
// one peer copy when the block is whole rows, else a 2-D copy (UVA: peer access makes the pointer
// addressable, cudaMemcpy2DAsync with cudaMemcpyDefault moves it over NVLink).
cudaError_t cudaMemcpy2DPeerAsync_compat(int32_t* dst, int dst_dev, const int32_t* src, int64_t n, int64_t cols,
                                         int64_t rows, cudaStream_t st) {
    int src_dev = 0;
    cudaGetDevice(&src_dev);
    if (cols == n)
        return cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, static_cast<size_t>(rows * n) * 4, st);
    return cudaMemcpy2DAsync(dst, static_cast<size_t>(n) * 4, src, static_cast<size_t>(n) * 4, static_cast<size_t>(cols) * 4,
                             static_cast<size_t>(rows), cudaMemcpyDefault, st);
}

// ---------------------------------------------------------------- the pipeline
struct HostGemm {
    const uint8_t* a_host = nullptr;  // A rows on the host (k bytes each), or
    const uint8_t* a_dev = nullptr;   // device-resident A (lda_dev pitch)
    int64_t lda_dev = 0;
    const int8_t* b_host = nullptr;   // B rows on the host, or
    const int8_t* b_dev = nullptr;    // device-resident B (ldb_dev pitch; the multi-GPU replica)
    int64_t ldb_dev = 0;
    cudaEvent_t b_ready = nullptr;    // recorded once b_dev holds B (may be null)
    int32_t* c_host = nullptr;        // host C (may be null when only gathering), and/or
    int32_t* c_gather = nullptr;      // a device buffer (row pitch n) on device gather_dev: C rows
    int gather_dev = -1;              // are peer-copied there tile by tile (NVLink)
    bool a_pinned = false, b_pinned = false, c_pinned = false;
    int64_t m = 0, n = 0, k = 0;
    int mode = 0, kernel = 0;
};

std::vector<std::pair<int64_t, int64_t>> blocks_growing(int64_t total, int64_t first, int64_t full, int64_t align) {
    std::vector<std::pair<int64_t, int64_t>> out;
    int64_t at = 0, size = std::max<int64_t>(align, std::min(first, full));
    while (at < total) {
        const int64_t len = std::min(total - at, size);
        out.push_back({at, len});
        at += len;
        size = std::min(full, size * 2);
    }
    return out;
}

ngemm_status host_pipeline(const HostGemm& g) {
    const int64_t m = g.m, n = g.n, k = g.k;
    const int64_t kp = round_up(k, 16);
    const bool a_res = g.a_dev != nullptr, b_res = g.b_dev != nullptr;
    // tile grid: column blocks (B rows) x row blocks (A rows)
    const int64_t rfull = round_up((m + 7) / 8, 256), cfull = round_up((n + 3) / 4, 256);
    const auto rows = a_res ? blocks_growing(m, rfull, rfull, 256) : blocks_growing(m, 256, rfull, 256);
    std::vector<std::pair<int64_t, int64_t>> cols;
    if (b_res) {
        cols.push_back({0, n});  // B resident: full-width row tiles, contiguous C copies
    } else {
        // streamed A: pass 0 must out-produce A's arrival by enough C backlog to cover B_1's load
        // (w0 >= 5K/16: 1.25 bytes of C per byte of A)
        const int64_t w0 = a_res ? std::min<int64_t>(1024, cfull) : std::max<int64_t>(cfull, round_up(5 * k / 16, 256));
        int64_t at = 0;
        while (at < n) {
            const int64_t len = std::min(n - at, at == 0 ? w0 : cfull);
            cols.push_back({at, len});
            at += len;
        }
    }
    const int ti = static_cast<int>(rows.size()), tj = static_cast<int>(cols.size());
    const bool stage_in = (!a_res && !g.a_pinned) || (!b_res && !g.b_pinned);
    const bool stage_out = g.c_host != nullptr && !g.c_pinned;
    if ((stage_in || stage_out) && kp > static_cast<int64_t>(kSlotBytes)) return NGEMM_ERR_UNSUPPORTED;  // caller falls back

    const size_t a_bytes = a_res ? 0 : static_cast<size_t>(m * kp), b_bytes = b_res ? 0 : static_cast<size_t>(n * kp);
    const size_t c_bytes = static_cast<size_t>(m * n) * 4;
    const size_t b_off = round_up(static_cast<int64_t>(a_bytes), 256), c_off = b_off + round_up(b_bytes, 256);
    cudaStream_t sin = nullptr, scomp = nullptr, sout = nullptr;
    // events: A blocks [0, ti), B blocks [ti, ti + tj), C tiles [ti + tj, ti + tj + ti*tj), done
    std::vector<cudaEvent_t> ev(static_cast<size_t>(ti + tj + ti * tj + 1), nullptr);
    ngemm_status s = NGEMM_OK;
    std::mutex err_mu;
    auto ck = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess) {
            std::lock_guard<std::mutex> lk(err_mu);
            if (s == NGEMM_OK) s = fail(NGEMM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
        }
        return e == cudaSuccess;
    };
    ck(cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&scomp, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking), "stream");
    for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    std::vector<Slot> in_slots, out_slots;
    static const int nslots = [] {  // experiments: NGEMM_STAGE_SLOTS (read once)
        const char* e = std::getenv("NGEMM_STAGE_SLOTS");
        return e ? std::max(2, std::atoi(e)) : 8;
    }();
    if (s == NGEMM_OK && stage_in && !take_slots(nslots, in_slots)) s = fail(NGEMM_ERR_CUDA, "pinned staging allocation failed");
    if (s == NGEMM_OK && stage_out && !take_slots(nslots, out_slots)) s = fail(NGEMM_ERR_CUDA, "pinned staging allocation failed");
    uint8_t* buf = nullptr;
    if (s == NGEMM_OK) ck(dev_alloc(&buf, c_off + c_bytes, sin), "device allocation");
    int32_t* dc = buf ? reinterpret_cast<int32_t*>(buf + c_off) : nullptr;

    // ---- H2D of `nrows` host rows (k bytes each) into device rows of pitch kp
    size_t in_next = 0;
    auto h2d_rows = [&](uint8_t* dst, const void* src, int64_t nrows, bool pinned) {
        if (s != NGEMM_OK) return;
        if (pinned) {
            ck(copy_rows_h2d(dst, kp, src, k, nrows, sin), "H2D");
            return;
        }
        const int64_t per = std::max<int64_t>(1, static_cast<int64_t>(kSlotBytes) / k);
        for (int64_t r = 0; r < nrows && s == NGEMM_OK; r += per) {
            const int64_t cnt = std::min(per, nrows - r);
            Slot& sl = in_slots[in_next++ % in_slots.size()];
            ck(cudaEventSynchronize(sl.ev), "staging wait");  // the slot's previous DMA is done
            par_copy_2d(sl.p, k, static_cast<const uint8_t*>(src) + r * k, k, k, cnt);
            ck(cudaMemcpy2DAsync(dst + r * kp, kp, sl.p, k, k, cnt, cudaMemcpyHostToDevice, sin), "H2D staged");
            ck(cudaEventRecord(sl.ev, sin), "record");
        }
    };

    // ---- output side: pageable C drains on its own thread, tile by tile in issue order
    std::mutex tmu;
    std::condition_variable tcv;
    int tiles_issued = 0;  // tile events recorded so far (by the issuing thread)
    bool abort_out = false;
    // the drain thread keeps its own status (the library's error message is thread-local, and the
    // issuing thread reads `s` without a lock); it is merged after the join
    std::atomic<bool> out_failed{false};
    std::string out_msg;
    std::thread out_thread;
    int dev_main = 0;
    cudaGetDevice(&dev_main);
    if (stage_out && s == NGEMM_OK) {
        out_thread = std::thread([&] {
            cudaSetDevice(dev_main);  // a new thread starts on device 0; the streams and events are dev_main's
            auto ck = [&](cudaError_t e, const char* what) {
                if (e != cudaSuccess && !out_failed.exchange(true)) out_msg = std::string(what) + ": " + cudaGetErrorString(e);
                return e == cudaSuccess;
            };
            struct Pending {
                Slot* sl;
                int64_t r0, c0, nr, nc;
            };
            std::deque<Pending> q;
            size_t next = 0;
            auto drain_one = [&] {
                Pending p = q.front();
                q.pop_front();
                if (!ck(cudaEventSynchronize(p.sl->ev), "D2H wait")) return;
                par_copy_2d(g.c_host + p.r0 * n + p.c0, n * 4, p.sl->p, p.nc * 4, p.nc * 4, p.nr);
            };
            int t = 0;
            for (int j = 0; j < tj; ++j)
                for (int i = 0; i < ti; ++i, ++t) {
                    {
                        std::unique_lock<std::mutex> lk(tmu);
                        tcv.wait(lk, [&] { return tiles_issued > t || abort_out; });
                        if (out_failed.load()) abort_out = true;
                        if (abort_out && tiles_issued <= t) {
                            while (!q.empty()) q.pop_front();
                            return;
                        }
                    }
                    const int64_t r0 = rows[i].first, nrows = rows[i].second;
                    const int64_t c0 = cols[j].first, ncols = cols[j].second;
                    ck(cudaStreamWaitEvent(sout, ev[ti + tj + t], 0), "wait");
                    const int64_t per = std::max<int64_t>(1, static_cast<int64_t>(kSlotBytes) / (ncols * 4));
                    for (int64_t r = 0; r < nrows; r += per) {
                        if (q.size() == out_slots.size()) drain_one();
                        Slot& sl = out_slots[next++ % out_slots.size()];
                        const int64_t cnt = std::min(per, nrows - r);
                        ck(cudaMemcpy2DAsync(sl.p, ncols * 4, dc + (r0 + r) * n + c0, n * 4, ncols * 4, cnt,
                                             cudaMemcpyDeviceToHost, sout), "D2H staged");
                        ck(cudaEventRecord(sl.ev, sout), "record");
                        q.push_back({&sl, r0 + r, c0, cnt, ncols});
                    }
                }
            while (!q.empty()) drain_one();
        });
    }

    // ---- issue: copies in first-use order, GEMMs, and (pinned C) the copies out
    if (s == NGEMM_OK) {
        int t = 0;
        for (int j = 0; j < tj; ++j) {
            const int64_t c0 = cols[j].first, ncols = cols[j].second;
            for (int i = 0; i < ti; ++i, ++t) {
                const int64_t r0 = rows[i].first, nrows = rows[i].second;
                if (s == NGEMM_OK && i == 0 && !b_res) {
                    h2d_rows(buf + b_off + c0 * kp, g.b_host + c0 * k, ncols, g.b_pinned);
                    ck(cudaEventRecord(ev[ti + j], sin), "record");
                }
                if (s == NGEMM_OK && t == 0 && b_res && g.b_ready) ck(cudaStreamWaitEvent(scomp, g.b_ready, 0), "wait");
                if (s == NGEMM_OK && j == 0 && !a_res) {
                    h2d_rows(buf + r0 * kp, g.a_host + r0 * k, nrows, g.a_pinned);
                    ck(cudaEventRecord(ev[i], sin), "record");
                }
                if (s == NGEMM_OK) {
                    if (!a_res) ck(cudaStreamWaitEvent(scomp, ev[i], 0), "wait");
                    if (!b_res) ck(cudaStreamWaitEvent(scomp, ev[ti + j], 0), "wait");
                }
                if (s == NGEMM_OK) {
                    const uint8_t* ablk = a_res ? g.a_dev + r0 * g.lda_dev : buf + r0 * kp;
                    const int64_t lda = a_res ? g.lda_dev : kp;
                    const int8_t* bblk = b_res ? g.b_dev + c0 * g.ldb_dev : reinterpret_cast<const int8_t*>(buf + b_off + c0 * kp);
                    const int64_t ldb = b_res ? g.ldb_dev : kp;
                    ngemm_status gs = run_gemm(ablk, lda, bblk, ldb, dc + r0 * n + c0, n, nrows, ncols, k, g.mode, g.kernel,
                                               scomp);
                    if (gs != NGEMM_OK) {
                        std::lock_guard<std::mutex> lk(err_mu);
                        if (s == NGEMM_OK) s = gs;
                    }
                }
                cudaEvent_t ev_c = ev[ti + tj + t];
                if (s == NGEMM_OK) ck(cudaEventRecord(ev_c, scomp), "record");
                if (s == NGEMM_OK && g.c_gather) {  // C rows assembled on the gather device (NVLink peer copy)
                    ck(cudaStreamWaitEvent(sout, ev_c, 0), "wait");
                    ck(cudaMemcpy2DPeerAsync_compat(g.c_gather + r0 * n + c0, g.gather_dev, dc + r0 * n + c0, n, ncols,
                                                    nrows, sout), "peer gather");
                }
                if (s == NGEMM_OK && g.c_host && !stage_out) {
                    ck(cudaStreamWaitEvent(sout, ev_c, 0), "wait");
                    if (tj == 1)
                        ck(cudaMemcpyAsync(g.c_host + r0 * n, dc + r0 * n, static_cast<size_t>(nrows * n) * 4,
                                           cudaMemcpyDeviceToHost, sout), "D2H C");
                    else
                        ck(cudaMemcpy2DAsync(g.c_host + r0 * n + c0, static_cast<size_t>(n) * 4, dc + r0 * n + c0,
                                             static_cast<size_t>(n) * 4, static_cast<size_t>(ncols) * 4,
                                             static_cast<size_t>(nrows), cudaMemcpyDeviceToHost, sout), "D2H C");
                }
                if (s != NGEMM_OK) break;
                {
                    std::lock_guard<std::mutex> lk(tmu);
                    tiles_issued = t + 1;
                }
                tcv.notify_all();
            }
            if (s != NGEMM_OK) break;
        }
    }
    {
        std::lock_guard<std::mutex> lk(tmu);
        abort_out = true;
    }
    tcv.notify_all();
    if (out_thread.joinable()) out_thread.join();
    if (out_failed.load() && s == NGEMM_OK) s = fail(NGEMM_ERR_CUDA, out_msg);
    if (buf) {
        cudaEvent_t ev_done = ev.back();
        ck(cudaEventRecord(ev_done, sout), "record");
        cudaStreamWaitEvent(sin, ev_done, 0);
        cudaStreamWaitEvent(sin, ev[ti + tj + ti * tj - 1], 0);
        cudaFreeAsync(buf, sin);
    }
    if (sin) ck(cudaStreamSynchronize(sin), "sync");
    if (sout) ck(cudaStreamSynchronize(sout), "sync");
    if (scomp) ck(cudaStreamSynchronize(scomp), "sync");
    give_slots(in_slots);
    give_slots(out_slots);
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    if (sin) cudaStreamDestroy(sin);
    if (scomp) cudaStreamDestroy(scomp);
    if (sout) cudaStreamDestroy(sout);
    return s;
}

// Large enough for the pipeline to pay (C >= 32 MiB and more than one tile row of work).
bool pipeline_worth(int64_t m, int64_t n, int64_t k) {
    return m >= 512 && n >= 256 && static_cast<double>(m) * n * 4 >= 32.0 * (1 << 20) && k <= (1 << 22);
}

}  // namespace

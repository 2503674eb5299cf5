// transfer.cu -- host -> HBM transfer of record columns, block-compressed on the way.
//
// The host-buffer entry points (heteff_analyze_host / _csr) are bound by PCIe (~55 GB/s
// on the B200 box: 17 B per interval at C5 is 34 GB per call).  Timestamps of a trace are
// dense: inside a block of kBlock records, starts sit within a short span and durations
// are small.  So the columns cross PCIe as
//
//   per block:  s0 = min start, widths ws / wd (1, 2 or 4 bytes; 8 = raw), then
//               start - s0 (ws bytes each) | end - start (wd bytes each) | kind (1 byte each)
//
// (raw 8-byte starts / ends when a span or a duration does not fit 32 bits, or an end
// precedes its start), encoded by host threads into pinned staging slots, copied, and
// expanded into the full u64 / u8 columns in HBM by a decode kernel -- exact for every
// input.  Host encoding (the columns read once from memory, ~110 GB/s on the box's 16
// cores), the copies and the decode run as a pipeline over chunks of kChunk records.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "transfer.cuh"

namespace hb {
namespace xfer {

// the block format (kBlock, BlockHdr) and the host encoder live in transfer.cuh /
// transfer_enc.cpp (compiled for AVX-512 when the host has it)
// one CTA per block: expand into the HBM columns.  Gap blocks rebuild their starts with a
// block-wide inclusive scan (16 consecutive records per thread, 64-bit sums).
__global__ void __launch_bounds__(256) decode_kernel(const uint8_t *__restrict__ chunk, uint64_t *__restrict__ S,
                                                     uint64_t *__restrict__ E, uint8_t *__restrict__ K)
{
    __shared__ uint64_t warp_tot[8];
    const BlockHdr h = reinterpret_cast<const BlockHdr *>(chunk + 16)[blockIdx.x];
    const int cnt = (int)h.cnt + 1;
    const int w = h.ws & 15;
    const uint8_t *ps = chunk + h.off;
    const uint8_t *pd = ps + ((cnt * w + 15) & ~15);
    const uint8_t *pk = pd + ((cnt * h.wd + 15) & ~15);
    const int64_t o = (int64_t)blockIdx.x * kBlock;
    auto field = [](const uint8_t *p, int wd, int i) -> uint64_t {
        switch (wd) {
            case 1: return p[i];
            case 2: return reinterpret_cast<const uint16_t *>(p)[i];
            case 4: return reinterpret_cast<const uint32_t *>(p)[i];
            default: return reinterpret_cast<const uint64_t *>(p)[i];
        }
    };
    if (h.ws & kDelta) {
        constexpr int kPer = kBlock / 256;
        const int b = threadIdx.x * kPer;
        uint64_t v[kPer], run = 0;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            v[q] = b + q < cnt ? field(ps, w, b + q) : 0ull;
            run += v[q];
        }
        // exclusive prefix of the thread sums across the CTA
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        uint64_t inc = run;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t x = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += x;
        }
        if (lane == 31) warp_tot[warp] = inc;
        __syncthreads();
        uint64_t acc = h.s0 + inc - run;
        for (int q = 0; q < warp; ++q) acc += warp_tot[q];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int i = b + q;
            acc += v[q];
            if (i < cnt) {
                const uint64_t e = h.wd == 8 ? field(pd, 8, i) : acc + field(pd, h.wd, i);
                S[o + i] = acc;
                E[o + i] = e;
                K[o + i] = pk[i];
            }
        }
        return;
    }
    for (int i = threadIdx.x; i < cnt; i += 256) {
        const uint64_t s = w == 8 ? field(ps, 8, i) : h.s0 + field(ps, w, i);
        const uint64_t e = h.wd == 8 ? field(pd, 8, i) : s + field(pd, h.wd, i);
        S[o + i] = s;
        E[o + i] = e;
        K[o + i] = pk[i];
    }
}

}  // namespace xfer

struct Job {
    int side;
    int64_t r0, n;
};

// The pipeline: encoder threads fill free pinned slots; this thread copies each filled slot
// to its device twin and launches the decode, recording an event that frees the slot.
int transfer_columns(TransferCtx &tc, const TransferSide *sides, int nsides, int nthreads, cudaStream_t s,
                     std::string &err)
{
    using namespace xfer;
    std::vector<Job> jobs;
    for (int q = 0; q < nsides; ++q)
        for (int64_t r = 0; r < sides[q].count; r += kChunk)
            jobs.push_back({q, r, std::min<int64_t>(kChunk, sides[q].count - r)});
    if (jobs.empty()) return 0;
    const int nslots = std::max(4, 2 * nthreads);
    const size_t sb = slot_bytes();
    if (tc.slots < nslots) {
        if (tc.pinned) cudaFreeHost(tc.pinned);
        if (tc.dev) cudaFree(tc.dev);
        for (cudaEvent_t ev : tc.events) cudaEventDestroy(ev);
        tc.events.clear();
        tc.pinned = nullptr;
        tc.dev = nullptr;
        tc.slots = 0;
        if (cudaMallocHost(&tc.pinned, sb * nslots) != cudaSuccess) { err = "alloc pinned transfer slots"; return -1; }
        if (cudaMalloc(&tc.dev, sb * nslots) != cudaSuccess) { err = "alloc device transfer slots"; return -1; }
        tc.events.resize(nslots);
        for (auto &ev : tc.events) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        tc.slots = nslots;
    }
    uint8_t *pin = static_cast<uint8_t *>(tc.pinned);
    uint8_t *dev = static_cast<uint8_t *>(tc.dev);

    std::mutex mu;
    std::condition_variable cv_free, cv_ready;
    std::deque<int> free_slots;
    for (int i = 0; i < nslots; ++i) free_slots.push_back(i);
    struct Ready { int job, slot; size_t bytes; };
    std::deque<Ready> ready;
    std::atomic<int> next{0};
    bool abort = false;

    auto worker = [&]() {
        for (;;) {
            const int j = next.fetch_add(1);
            if (j >= (int)jobs.size()) return;
            int slot;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_free.wait(lk, [&] { return !free_slots.empty() || abort; });
                if (abort) return;
                slot = free_slots.front();
                free_slots.pop_front();
            }
            const Job &jb = jobs[j];
            const TransferSide &sd = sides[jb.side];
            const size_t bytes = encode_chunk(sd.start, sd.end, sd.kind, jb.r0, jb.n, pin + (size_t)slot * sb);
            {
                std::lock_guard<std::mutex> lk(mu);
                ready.push_back({j, slot, bytes});
            }
            cv_ready.notify_one();
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t) pool.emplace_back(worker);

    std::vector<int> inflight;   // slots with a copy / decode in flight
    int done = 0, rc = 0;
    while (done < (int)jobs.size()) {
        Ready r{};
        bool got = false;
        {
            std::unique_lock<std::mutex> lk(mu);
            cv_ready.wait_for(lk, std::chrono::microseconds(50), [&] { return !ready.empty(); });
            if (!ready.empty()) { r = ready.front(); ready.pop_front(); got = true; }
        }
        if (got) {
            const Job &jb = jobs[r.job];
            const TransferSide &sd = sides[jb.side];
            const int nb = (int)((jb.n + kBlock - 1) / kBlock);
            uint8_t *d = dev + (size_t)r.slot * sb;
            cudaError_t e = cudaMemcpyAsync(d, pin + (size_t)r.slot * sb, r.bytes, cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) {
                decode_kernel<<<nb, 256, 0, s>>>(d, sd.dst_start + jb.r0, sd.dst_end + jb.r0, sd.dst_kind + jb.r0);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaEventRecord(tc.events[r.slot], s);
            if (e != cudaSuccess) { err = cudaGetErrorString(e); rc = -1; break; }
            inflight.push_back(r.slot);
            ++done;
        }
        // slots whose copy has completed go back to the encoders
        for (size_t i = 0; i < inflight.size();) {
            if (cudaEventQuery(tc.events[inflight[i]]) == cudaSuccess) {
                {
                    std::lock_guard<std::mutex> lk(mu);
                    free_slots.push_back(inflight[i]);
                }
                cv_free.notify_one();
                inflight[i] = inflight.back();
                inflight.pop_back();
            } else {
                ++i;
            }
        }
    }
    if (rc != 0) {
        std::lock_guard<std::mutex> lk(mu);
        abort = true;
    }
    cv_free.notify_all();
    for (auto &t : pool) t.join();
    // on failure nothing after this call waits for the copies already issued: drain them
    // before the pinned slots can be reused (on success the caller's analysis syncs the stream)
    if (rc != 0) cudaStreamSynchronize(s);
    cudaGetLastError();
    return rc;
}

void transfer_free(TransferCtx &tc)
{
    if (tc.pinned) cudaFreeHost(tc.pinned);
    if (tc.dev) cudaFree(tc.dev);
    for (cudaEvent_t ev : tc.events) cudaEventDestroy(ev);
    tc.events.clear();
    tc.pinned = tc.dev = nullptr;
    tc.slots = 0;
}

}  // namespace hb

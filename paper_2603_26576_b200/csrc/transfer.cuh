// transfer.cuh -- block-compressed host -> HBM transfer of record columns (transfer.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace hb {

namespace xfer {
constexpr int kBlock = 4096;                       // records per block
constexpr int kBlocksPerChunk = 256;               // 1 Mi records per chunk
constexpr int64_t kChunk = (int64_t)kBlock * kBlocksPerChunk;

constexpr uint8_t kDelta = 16;   // BlockHdr::ws flag: starts stored as gaps to the previous start

struct BlockHdr {           // 16 bytes, in the chunk's block table
    uint64_t s0;            // min start (the first one for gap blocks; 0 for raw starts)
    uint32_t off;           // payload offset from the chunk start (16-byte aligned)
    uint8_t ws, wd;         // widths: 1, 2, 4, or 8 (raw values); ws | kDelta: gaps
    uint16_t cnt;           // records in the block - 1 (<= 4095)
};
static_assert(sizeof(BlockHdr) == 16, "block header");

// worst case bytes of one encoded chunk
inline size_t slot_bytes() { return 16 + (size_t)kBlocksPerChunk * (sizeof(BlockHdr) + (size_t)kBlock * 17 + 48); }

// encode records [r0, r0 + n) of one side (n <= kChunk) into `out`; returns the bytes used
size_t encode_chunk(const uint64_t *S, const uint64_t *E, const uint8_t *K, int64_t r0, int64_t n, uint8_t *out);
}  // namespace xfer

// pinned staging slots + their device twins, cached in the engine context
struct TransferCtx {
    void *pinned = nullptr;
    void *dev = nullptr;
    int slots = 0;
    std::vector<cudaEvent_t> events;
};

// one record set: host columns in, HBM columns out
struct TransferSide {
    const uint64_t *start, *end;
    const uint8_t *kind;
    int64_t count;
    uint64_t *dst_start, *dst_end;
    uint8_t *dst_kind;
};

// encode on `nthreads` host threads, copy and decode on stream `s`; returns 0 or -1 (err set).
// When it returns, every copy and decode is enqueued on `s` (the caller orders its kernels after).
int transfer_columns(TransferCtx &tc, const TransferSide *sides, int nsides, int nthreads, cudaStream_t s,
                     std::string &err);
void transfer_free(TransferCtx &tc);

}  // namespace hb

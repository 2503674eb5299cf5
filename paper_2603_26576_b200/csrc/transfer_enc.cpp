// transfer_enc.cpp -- host encoder of the block-compressed column transfer (transfer.cu).
// Plain C++ (compiled by the host compiler): the hot loops are written for the vectorizer
// and compiled twice, generic and for AVX-512, picked at run time.
#include <algorithm>
#include <cstdint>
#include <cstring>

#include "transfer.cuh"

namespace hb {
namespace xfer {

static inline uint8_t width_of(uint64_t v) { return v < 256 ? 1 : v < 65536 ? 2 : v <= 0xffffffffull ? 4 : 8; }
static inline size_t up16(size_t x) { return (x + 15) & ~(size_t)15; }

template <typename T>
static inline __attribute__((always_inline)) void put_off(uint8_t *dst, const uint64_t *__restrict__ v, uint64_t base,
                                                          int n)
{
    T *__restrict__ o = reinterpret_cast<T *>(dst);
    for (int i = 0; i < n; ++i) o[i] = (T)(v[i] - base);
}

template <typename T>
static inline __attribute__((always_inline)) void put_gap(uint8_t *dst, const uint64_t *__restrict__ v, int n)
{
    T *__restrict__ o = reinterpret_cast<T *>(dst);
    o[0] = 0;
    for (int i = 1; i < n; ++i) o[i] = (T)(v[i] - v[i - 1]);
}

template <typename T>
static inline __attribute__((always_inline)) void put_dur(uint8_t *dst, const uint64_t *__restrict__ s,
                                                          const uint64_t *__restrict__ e, int n)
{
    T *__restrict__ o = reinterpret_cast<T *>(dst);
    for (int i = 0; i < n; ++i) o[i] = (T)(e[i] - s[i]);
}

static inline __attribute__((always_inline)) size_t encode_body(const uint64_t *S, const uint64_t *E,
                                                                const uint8_t *K, int64_t r0, int64_t n,
                                                                uint8_t *out)
{
    const int nb = (int)((n + kBlock - 1) / kBlock);
    reinterpret_cast<uint32_t *>(out)[0] = (uint32_t)nb;
    BlockHdr *tab = reinterpret_cast<BlockHdr *>(out + 16);
    size_t pos = up16(16 + (size_t)nb * sizeof(BlockHdr));
    for (int b = 0; b < nb; ++b) {
        const int64_t i0 = r0 + (int64_t)b * kBlock;
        const int cnt = (int)std::min<int64_t>(kBlock, r0 + n - i0);
        const uint64_t *__restrict__ s = S + i0;
        const uint64_t *__restrict__ e = E + i0;
        // reductions over the block (it stays in L1 / L2 for the writes below)
        uint64_t mn = ~0ull, mx = 0, dmax = 0, neg = 0, down = 0, gmax = 0;
        for (int i = 0; i < cnt; ++i) {
            mn = std::min(mn, s[i]);
            mx = std::max(mx, s[i]);
        }
        for (int i = 0; i < cnt; ++i) {
            neg |= (uint64_t)(e[i] < s[i]);
            dmax = std::max(dmax, e[i] - s[i]);
        }
        for (int i = 1; i < cnt; ++i) {   // start-sorted blocks: the gaps between starts
            down |= (uint64_t)(s[i] < s[i - 1]);
            gmax = std::max(gmax, s[i] - s[i - 1]);
        }
        BlockHdr h;
        const uint8_t wo = width_of(mx - mn), wg = down ? 8 : width_of(gmax);
        const bool delta = wg < wo;   // gaps narrower than offsets: starts as gaps (decoded by a scan)
        h.ws = delta ? (uint8_t)(wg | kDelta) : wo;
        h.wd = neg ? 8 : width_of(dmax);
        h.s0 = wo == 8 && !delta ? 0 : mn;   // delta blocks are sorted: mn is the first start
        h.cnt = (uint16_t)(cnt - 1);
        h.off = (uint32_t)pos;
        uint8_t *p = out + pos;
        const int w = h.ws & 15;
        if (delta) {
            switch (w) {
                case 1: put_gap<uint8_t>(p, s, cnt); break;
                case 2: put_gap<uint16_t>(p, s, cnt); break;
                default: put_gap<uint32_t>(p, s, cnt); break;
            }
        } else {
            switch (w) {
                case 1: put_off<uint8_t>(p, s, mn, cnt); break;
                case 2: put_off<uint16_t>(p, s, mn, cnt); break;
                case 4: put_off<uint32_t>(p, s, mn, cnt); break;
                default: memcpy(p, s, (size_t)cnt * 8);
            }
        }
        p += up16((size_t)cnt * w);
        switch (h.wd) {
            case 1: put_dur<uint8_t>(p, s, e, cnt); break;
            case 2: put_dur<uint16_t>(p, s, e, cnt); break;
            case 4: put_dur<uint32_t>(p, s, e, cnt); break;
            default: memcpy(p, e, (size_t)cnt * 8);   // raw ends
        }
        p += up16((size_t)cnt * h.wd);
        memcpy(p, K + i0, (size_t)cnt);
        p += up16((size_t)cnt);
        pos = (size_t)(p - out);
        tab[b] = h;
    }
    return pos;
}

__attribute__((target("avx512f,avx512bw,avx512vl,avx512dq"))) static size_t
encode_avx512(const uint64_t *S, const uint64_t *E, const uint8_t *K, int64_t r0, int64_t n, uint8_t *out)
{
    return encode_body(S, E, K, r0, n, out);
}

static size_t encode_generic(const uint64_t *S, const uint64_t *E, const uint8_t *K, int64_t r0, int64_t n,
                             uint8_t *out)
{
    return encode_body(S, E, K, r0, n, out);
}

size_t encode_chunk(const uint64_t *S, const uint64_t *E, const uint8_t *K, int64_t r0, int64_t n, uint8_t *out)
{
    static const bool avx512 = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                               __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512dq");
    return avx512 ? encode_avx512(S, E, K, r0, n, out) : encode_generic(S, E, K, r0, n, out);
}

}  // namespace xfer
}  // namespace hb

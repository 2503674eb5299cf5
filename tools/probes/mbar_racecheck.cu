// Does compute-sanitizer racecheck model mbarrier arrive (release) / wait (acquire)?
//
// The engine's producer warp fills shared memory with generic stores, arrives on a
// "full" mbarrier; the compute warps wait on it, read, arrive on "empty"; the producer
// waits on "empty" before refilling.  This probe is that protocol and nothing else:
// one producer warp, two consumer warps, a 2-stage ring, 64 rounds.  It is correct by
// the PTX memory model (mbarrier.arrive has release, mbarrier.try_wait acquire
// semantics at CTA scope); the host side checks every consumed value.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2603_26576_b200/csrc \
//        tools/probes/mbar_racecheck.cu -o /tmp/mbar_probe
//   compute-sanitizer --tool racecheck /tmp/mbar_probe
#include <cstdio>
#include <cstdint>
#include "engine.cuh"
#include "ptx.cuh"

using namespace hb;

constexpr int kStagesP = 2, kWords = 512, kRounds = 64, kConsumers = 2;

__global__ void probe(unsigned long long *out)
{
    __shared__ uint64_t full[kStagesP], empty[kStagesP];
    __shared__ int buf[kStagesP][kWords];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesP; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kConsumers); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {                       // producer
        for (int it = 0; it < kRounds; ++it) {
            const int st = it % kStagesP;
            if (it >= kStagesP) mbar_wait(&empty[st], (uint32_t)(((it / kStagesP) - 1) & 1));
            for (int i = lane; i < kWords; i += 32) buf[st][i] = it * kWords + i;   // generic stores
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[st]);
        }
    } else {                               // consumers
        unsigned long long acc = 0;
        for (int it = 0; it < kRounds; ++it) {
            const int st = it % kStagesP;
            mbar_wait(&full[st], (uint32_t)((it / kStagesP) & 1));
            for (int i = lane; i < kWords; i += 32) acc += (unsigned long long)buf[st][i];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        atomicAdd(out, acc);
    }
}

int main()
{
    unsigned long long *d, h = 0;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    probe<<<1, 32 * (1 + kConsumers)>>>(d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const unsigned long long n = (unsigned long long)kRounds * kWords;
    const unsigned long long want = kConsumers * (n * (n - 1) / 2);
    printf("mbarrier probe: sum %llu, expected %llu -> %s\n", h, want, h == want ? "ok" : "WRONG");
    return h == want ? 0 : 1;
}

// peer.cuh — the direct-store halo transport: the boundary launch of the skewed schedule
// writes the (u^{j+1}, p^{j+2}) of every block a peer rank reads straight into that peer's ghost rows
// (peer memory: CUDA IPC over NVLink on a multi-GPU box, another volume's workspace in one process), and a
// per-peer counter in the peer's memory says "iteration done".  Shared by iterate.cu (the fused epilogue of
// k_skew) and shard.cu (push / signal / wait kernels, host orchestration).
#pragma once

#include <stdint.h>

namespace hvg {

constexpr int kMaxDst = 4;   // peers one boundary block is written to (route partition: at most 2)

// Field buffers of one peer, as mapped into this process.
struct PeerOut {
    float *u[2];                  // the peer's u (index 0) and second u buffer (index 1)
    float *ub[2];                 // the peer's ū buffers (the prologue exchange)
    float *px[2], *py[2], *pz[2];
    unsigned long long *flags;    // the peer's arrival counters, one per source rank
};

// Destinations of one boundary row: (peer slot, row in that peer's store), slot −1 ends the list.
struct PeerDst {
    int32_t slot[kMaxDst];
    int32_t row[kMaxDst];
};

}  // namespace hvg

// shard.h — route-axis spatial sharding: host-side shard plan and the sharded
// runtime hooks used by vol_api.cu.  Not part of the C ABI.
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/vol.h"
#include "internal.h"

struct vol_s;

namespace hvg {

// Plan of one rank.  Store rows: [0, n_local) are the rank's blocks in global order, then the
// ghost blocks (remote blocks whose data the rank reads), grouped by owner rank, ascending global
// index inside a group (= the order in which that owner sends them).
struct ShardPlan {
    int rank = 0, world = 1;
    std::vector<int64_t> local;        // global index of store row r < n_local (launch A rows, then B rows)
    std::vector<int32_t> local_caller; // position of store row r among the rank's blocks in global order
    int64_t nA = 0;                    // rows [0, nA): no remote neighbour (launch A); [nA, n_local): launch B
    std::vector<int64_t> ghost;        // global index of store row n_local + k
    std::vector<int64_t> recv_off, recv_cnt;  // [world] slice of `ghost` received from each peer
    std::vector<int64_t> send_rows;    // local store rows sent, grouped by peer (rank order), peer's recv order
    std::vector<int64_t> send_off, send_cnt;  // [world] slice of send_rows per peer
    std::string error;
    uint64_t digest = 0;               // digest of the plan's inputs (coordinates, owner map) when known, else 0
    // row maps of the store (filled with the cached plan): global index of store row r (local, then ghost
    // rows) and the store row of every global block (−1: not held)
    std::vector<int64_t> rows;
    std::vector<int32_t> store_of_global;
    int64_t n_local() const { return (int64_t)local.size(); }
    int64_t n_ghost() const { return (int64_t)ghost.size(); }
};

// Computes rank `rank`'s plan from the global block coordinates and owner map (host only).
bool make_shard_plan(const int32_t *xyz, int64_t n_global, const int32_t *part, int world, int rank, ShardPlan &plan);

// Morton order of the given global blocks: rows[k] = position (in `global_of_row`) of the k-th block.
void morton_sort_rows(const int32_t *xyz, const std::vector<int64_t> &global_of_row, std::vector<int32_t> &rows);

size_t shard_extra_bytes(const ShardPlan &plan);

}  // namespace hvg

// runtime hooks (shard.cu)
struct ShardRuntime;
vol_status shard_setup(vol_s *v, const hvg::ShardPlan &plan, const vol_dist *dist);
vol_status shard_after_create(vol_s *v);
vol_status shard_reset(vol_s *v);
vol_status shard_iterate(vol_s *v, const hvg::IterParams &P, int32_t iters);
vol_status shard_timing(vol_s *v, float *interior_ms, float *exchange_ms, float *boundary_ms);
vol_status shard_refresh_for_energy(vol_s *v);
vol_status shard_allreduce_energy(vol_s *v, double *d_eout);
void shard_destroy(vol_s *v);

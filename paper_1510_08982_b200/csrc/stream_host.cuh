// stream_host.cuh -- host side of K5 (async_stream.cuh): layout of the ring
// state, PE link descriptors (local rings, device-boundary receive rings),
// seeding and launches.  Used by the single-GPU entry points and by the
// multi-GPU slab API (heat_plan_xlink_*).
#pragma once

#include <functional>
#include <vector>

#include "async_stream.cuh"
#include "runtime.cuh"

namespace hb {

// How a slab meets other devices.  On one device everything is local; a
// multi-GPU rank has external neighbours whose receive rings it writes with
// P2P stores (pointers opened through CUDA IPC).
struct StreamExternal {
    bool left = false, right = false;  // slab end borders another device
    double* left_push_ring = nullptr;  // left device's receive ring for its RIGHT neighbour
    unsigned long long* left_push_prog = nullptr;
    double* right_push_ring = nullptr;  // right device's receive ring for its LEFT neighbour
    unsigned long long* right_push_prog = nullptr;
    long long pe_offset = 0;  // global index of local PE 0
    long long P_global = 0;   // 0 = this launch holds the whole domain
};

// Device scratch of one streaming run (rings persist across its launches).
struct StreamLayout {
    size_t P = 0, Tp = 0;
    int R = 0, D = 0;
    int G = 1;  // device groups inside this launch (> 1: emulated device boundaries)
    int V = 32; // points per lane of the stream kernel for this layout (48 or 32)
    int H = 32; // halo points per side = steps per pass (64 or 32)
    size_t o_ringL, o_ringR, o_progL, o_progR, o_recvL, o_recvR, o_rprogL, o_rprogR, o_done,
        o_counter, o_offL, o_offR, o_gthr, o_stats, o_abort, o_links, o_seeds, bytes;
};

int stream_layout(const AsyncRunSpec& s, int groups, const StreamExternal& ext, StreamLayout& L,
                  std::vector<int>& offL, std::vector<int>& offR);

// Optional K5 logs (AsyncStreamArgs::edge_log / used_log), device memory.
struct StreamLogs {
    double* edge_log = nullptr;
    int* used_log = nullptr;
};

// Advances bufs[cur] by `steps` from absolute step k0; init=true seeds the
// local rings and the in-launch receive rings and uploads the tables.
int async_stream_advance(int sms, cudaStream_t st, double* bufs[2], int& cur, const AsyncRunSpec& s,
                         const StreamLayout& L, char* base, const StreamExternal& ext,
                         const std::vector<int>& offL, const std::vector<int>& offR, size_t k0,
                         size_t steps, bool init, unsigned int* flag, float* device_ms,
                         const StreamLogs* logs = nullptr);

// Step-0 values this slab owes its external neighbours (P2P stores).
int stream_seed_external(cudaStream_t st, const double* field, const AsyncRunSpec& s,
                         const StreamExternal& ext);

// Whole-run driver used by heat_async_run / heat_exec_run for wide PEs.
int async_stream_run(DevCtx& d, const AsyncRunSpec& s, double* bufs[2], int& cur, size_t stride,
                     const std::function<int(size_t, const double*)>& on_record,
                     unsigned long long* host_stats, float* device_ms,
                     const StreamLogs* logs = nullptr);

// HEAT_VIRTUAL_DEVICES=G splits a single-GPU run into G device groups whose
// boundaries go through the cross-device (system-scope receive ring) path.
int virtual_device_groups(size_t P);

}  // namespace hb

// stream_host.cu -- K5 host code: ring layout, PE link descriptors, seeding,
// launches (see stream_host.cuh, async_stream.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "stream_host.cuh"

namespace hb {

namespace {

// Tile geometry (points per lane V, halo H = steps per pass) of the stream
// kernel for PEs of n points: the first of 48x64, 48x32, 32x32 under which
// a PE spans >= 2 tiles and its last tile holds >= H points (an interior
// tile's window must not reach into the next PE).  HEAT_ASYNC_GEOMETRY
// ("48x64", "48x32", "32x32") forces one where it fits, for A/B.
void stream_geometry(size_t n, int& V, int& H) {
    static const int forced = [] {
        const char* e = std::getenv("HEAT_ASYNC_GEOMETRY");
        if (!e) return 0;
        const std::string g(e);
        return g == "48x64" ? 1 : g == "48x32" ? 2 : g == "32x32" ? 3 : 0;
    }();
    const struct { int V, H; long long out; } cand[3] = {
        {48, 64, SyncTB<double, 48, 64>::kOut},
        {48, 32, SyncTB<double, 48, 32>::kOut},
        {32, 32, SyncTB<double, 32, 32>::kOut}};
    for (int i = forced ? forced - 1 : 0; i < 3; ++i) {
        const long long rem = (long long)n % cand[i].out;
        if ((long long)n > cand[i].out && (rem == 0 || rem >= cand[i].H)) {
            V = cand[i].V;
            H = cand[i].H;
            return;
        }
    }
    V = H = 32;
}
// Done-signals deferred per release fence (HEAT_K5_PEND, for A/B).
int env_int(const char* name, int dflt, int lo, int hi) {
    const char* e = std::getenv(name);
    if (!e || !*e) return dflt;
    return std::min(hi, std::max(lo, std::atoi(e)));
}
int stream_pend_max() {
    static const int v = env_int("HEAT_K5_PEND", 2, 1, kMaxPend);
    return v;
}
constexpr int kSU = 32;  // tensor-map unit (points); PEs are whole units

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// ring[0] = field[src] (the step-0 edge value), prog = 0
struct SeedOp {
    double* ring;
    unsigned long long* prog;
    long long src;
    int sys;  // the ring lives on another device
};

__global__ void stream_seed_kernel(const double* __restrict__ field, const SeedOp* ops, int nops) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nops; i += gridDim.x * blockDim.x) {
        const SeedOp o = ops[i];
        if (o.sys) {
            st_relaxed_sys_f64(o.ring, field[o.src]);
            st_release_sys(reinterpret_cast<uint64_t*>(o.prog), 0);
        } else {
            o.ring[0] = field[o.src];
            *o.prog = 0;
        }
    }
}

// `dev` (capacity `cap` ops) is a persistent device table, e.g. in the run's
// scratch; without one a temporary is allocated and the call synchronises.
// (A pageable-source cudaMemcpyAsync has taken its copy when it returns, so
// the host vector may go either way.)
int launch_seed(cudaStream_t st, const double* field, const std::vector<SeedOp>& ops,
                SeedOp* dev = nullptr, size_t cap = 0) {
    if (ops.empty()) return HEAT_OK;
    const bool tmp = dev == nullptr || ops.size() > cap;
    SeedOp* d_ops = dev;
    if (tmp) HB_CUDA(cudaMallocAsync(&d_ops, ops.size() * sizeof(SeedOp), st));
    HB_CUDA(cudaMemcpyAsync(d_ops, ops.data(), ops.size() * sizeof(SeedOp), cudaMemcpyHostToDevice,
                            st));
    stream_seed_kernel<<<int(std::min<size_t>(1024, (ops.size() + 255) / 256)), 256, 0, st>>>(
        field, d_ops, int(ops.size()));
    HB_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (tmp) {
        HB_CUDA(cudaFreeAsync(d_ops, st));
        HB_CUDA(cudaStreamSynchronize(st));
    }
    return HEAT_OK;
}

template <typename T>
T* at(char* base, size_t off) {
    return reinterpret_cast<T*>(base + off);
}

// Global neighbour of global PE gp (-1: none at a Dirichlet end).
long long left_of(long long gp, long long Pg, bool dir) { return gp > 0 ? gp - 1 : (dir ? -1 : Pg - 1); }
long long right_of(long long gp, long long Pg, bool dir) { return gp + 1 < Pg ? gp + 1 : (dir ? -1 : 0); }

void build_links(const StreamLayout& L, char* base, const AsyncRunSpec& s, const StreamExternal& ext,
                 std::vector<PeLink>& links, std::vector<SeedOp>& seeds, int& pin_first,
                 int& pin_last) {
    const long long P = (long long)L.P, Pv = P / L.G, R = L.R;
    const long long Pg = ext.P_global > 0 ? ext.P_global : P;
    const bool dir = s.bc_kind == HEAT_BC_DIRICHLET;
    double* ringL = at<double>(base, L.o_ringL);
    double* ringR = at<double>(base, L.o_ringR);
    auto* progL = at<unsigned long long>(base, L.o_progL);
    auto* progR = at<unsigned long long>(base, L.o_progR);
    double* recvL = at<double>(base, L.o_recvL);
    double* recvR = at<double>(base, L.o_recvR);
    auto* rprogL = at<unsigned long long>(base, L.o_rprogL);
    auto* rprogR = at<unsigned long long>(base, L.o_rprogR);
    links.assign(size_t(P), PeLink{});
    pin_first = pin_last = -1;
    const long long n = (long long)s.n;
    for (long long p = 0; p < P; ++p) {
        PeLink& lk = links[size_t(p)];
        const long long gp = ext.pe_offset + p, g = p / Pv;
        if (dir && gp == 0) pin_first = int(p);
        if (dir && gp == Pg - 1) pin_last = int(p);
        lk.pubF[0] = ringL + p * R;
        lk.pubF_prog[0] = progL + p;
        lk.pubL[0] = ringR + p * R;
        lk.pubL_prog[0] = progR + p;
        seeds.push_back({ringL + p * R, progL + p, p * n, 0});
        seeds.push_back({ringR + p * R, progR + p, p * n + n - 1, 0});
        // left neighbour
        const long long gl = left_of(gp, Pg, dir);
        if (gl >= 0) {
            const long long pl = gl - ext.pe_offset;
            const bool in_launch = pl >= 0 && pl < P;
            if (in_launch && pl / Pv == g) {  // same device: local rings
                lk.srcL = ringR + pl * R;
                lk.progL_src = progR + pl;
            } else {  // device boundary: read my receive ring
                lk.srcL = recvL + g * R;
                lk.progL_src = rprogL + g;
                lk.flags |= kLinkSrcLSys;
                if (in_launch) {  // emulated: the neighbour pushes into it, seeded here
                    links[size_t(pl)].pubL[1] = recvL + g * R;  // (filled again below if pl > p)
                    links[size_t(pl)].pubL_prog[1] = rprogL + g;
                    links[size_t(pl)].flags |= kLinkPubL1Sys;
                    seeds.push_back({recvL + g * R, rprogL + g, pl * n + n - 1, 0});
                } else {  // another rank: my first point goes to its receive ring
                    lk.pubF[1] = ext.left_push_ring;
                    lk.pubF_prog[1] = ext.left_push_prog;
                    lk.flags |= kLinkPubF1Sys;
                }
            }
        }
        // right neighbour
        const long long gr = right_of(gp, Pg, dir);
        if (gr >= 0) {
            const long long pr = gr - ext.pe_offset;
            const bool in_launch = pr >= 0 && pr < P;
            if (in_launch && pr / Pv == g) {
                lk.srcR = ringL + pr * R;
                lk.progR_src = progL + pr;
            } else {
                lk.srcR = recvR + g * R;
                lk.progR_src = rprogR + g;
                lk.flags |= kLinkSrcRSys;
                if (in_launch) {
                    links[size_t(pr)].pubF[1] = recvR + g * R;
                    links[size_t(pr)].pubF_prog[1] = rprogR + g;
                    links[size_t(pr)].flags |= kLinkPubF1Sys;
                    seeds.push_back({recvR + g * R, rprogR + g, pr * n, 0});
                } else {
                    lk.pubL[1] = ext.right_push_ring;
                    lk.pubL_prog[1] = ext.right_push_prog;
                    lk.flags |= kLinkPubL1Sys;
                }
            }
        }
    }
    // publish targets set for a neighbour processed earlier survive: a PE's
    // pubF[1]/pubL[1] are written only by its own device-boundary neighbours,
    // and the resets above only touch pub*[0].
}

}  // namespace

int heat_k5_geometry_query(size_t n, int* points_per_lane, int* halo) {
    int V = 32, H = 32;
    stream_geometry(n, V, H);
    if (points_per_lane) *points_per_lane = V;
    if (halo) *halo = H;
    return HEAT_OK;
}

int virtual_device_groups(size_t P) {
    const char* e = std::getenv("HEAT_VIRTUAL_DEVICES");
    if (!e) return 1;
    const int g = std::atoi(e);
    return (g >= 1 && P % size_t(g) == 0) ? g : 1;
}

int stream_layout(const AsyncRunSpec& s, int groups, const StreamExternal& ext, StreamLayout& L,
                  std::vector<int>& offL, std::vector<int>& offR) {
    if (s.n % kSU != 0)
        return fail(HEAT_EINVAL, "async: PEs wider than 1024 points must be a multiple of 32 points");
    L.P = s.N / s.n;
    stream_geometry(s.n, L.V, L.H);
    const long long tile_out = 32LL * L.V - 2LL * L.H;
    L.Tp = (s.n + tile_out - 1) / tile_out;
    if (L.Tp < 2) return fail(HEAT_ELOGIC, "async stream: a PE needs >= 2 tiles");
    L.G = (groups >= 1 && L.P % size_t(groups) == 0) ? groups : 1;
    L.R = 64;
    while (L.R < 2 * int(s.q) + 2) L.R *= 2;
    const bool dir = s.bc_kind == HEAT_BC_DIRICHLET;
    if (ext.P_global > 0) {  // draw ranks follow the global PE enumeration
        std::vector<int> gL, gR;
        L.D = draw_offsets(size_t(ext.P_global) * s.n, s.n, dir, gL, gR);
        offL.assign(gL.begin() + ext.pe_offset, gL.begin() + ext.pe_offset + L.P);
        offR.assign(gR.begin() + ext.pe_offset, gR.begin() + ext.pe_offset + L.P);
    } else {
        L.D = draw_offsets(s.N, s.n, dir, offL, offR);
    }
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += align256(b); return o; };
    L.o_ringL = take(L.P * L.R * sizeof(double));
    L.o_ringR = take(L.P * L.R * sizeof(double));
    L.o_progL = take(L.P * 8);
    L.o_progR = take(L.P * 8);
    L.o_recvL = take(size_t(L.G) * L.R * sizeof(double));
    L.o_recvR = take(size_t(L.G) * L.R * sizeof(double));
    L.o_rprogL = take(size_t(L.G) * 8);
    L.o_rprogR = take(size_t(L.G) * 8);
    L.o_done = take(L.P * L.Tp * 4);
    L.o_counter = take(8);
    L.o_offL = take(L.P * 4);
    L.o_offR = take(L.P * 4);
    L.o_gthr = take(std::max<size_t>(1, s.q - 1) * sizeof(uint64_t));
    L.o_stats = take(kStatWords * 8);
    L.o_abort = take(4);
    L.o_links = take(L.P * sizeof(PeLink));
    L.o_seeds = take((2 * L.P + 2 * size_t(L.G)) * sizeof(SeedOp));
    L.bytes = off;
    return HEAT_OK;
}

int stream_seed_external(cudaStream_t st, const double* field, const AsyncRunSpec& s,
                         const StreamExternal& ext) {
    std::vector<SeedOp> ops;
    const long long P = (long long)(s.N / s.n), n = (long long)s.n;
    if (ext.left && ext.left_push_ring) ops.push_back({ext.left_push_ring, ext.left_push_prog, 0, 1});
    if (ext.right && ext.right_push_ring)
        ops.push_back({ext.right_push_ring, ext.right_push_prog, P * n - 1, 1});
    return launch_seed(st, field, ops);
}

// Launch of the stream kernel with V-point lanes (tensor maps in 32-point units).
template <int V, int H>
int launch_stream(int sms, cudaStream_t st, double* const bufs[2], int cur, long long N,
                  const AsyncStreamArgs& a) {
    using T = SyncTB<double, V, H>;
    const int smem = T::smem_bytes(2);
    int per_sm = 0;  // per device: the persistent grid is every resident CTA
    HB_TRY(kernel_smem_config(reinterpret_cast<const void*>(async_stream_kernel<V, H>), smem,
                              T::kThreads, &per_sm));
    const long long nunits = N / T::kUnit;
    CUtensorMap ld[2], stm[2];
    for (int b = 0; b < 2; ++b) {
        HB_TRY(make_chunk_map_f64(&ld[b], bufs[b], nunits, T::kWinUnits));
        HB_TRY(make_chunk_map_f64(&stm[b], bufs[b], nunits, T::kOutUnits));
    }
    // maps follow the pass parity: pass pi reads a.buf[pi & 1]
    async_stream_kernel<V, H><<<sms * per_sm, T::kThreads, smem, st>>>(ld[cur], ld[cur ^ 1],
                                                                      stm[cur], stm[cur ^ 1], a);
    HB_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return HEAT_OK;
}

int async_stream_advance(int sms, cudaStream_t st, double* bufs[2], int& cur, const AsyncRunSpec& s,
                         const StreamLayout& L, char* base, const StreamExternal& ext,
                         const std::vector<int>& offL, const std::vector<int>& offR, size_t k0,
                         size_t steps, bool init, unsigned int* flag, float* device_ms,
                         const StreamLogs* logs) {
    // the pinned Dirichlet ends: global PE 0's first point, global PE Pg-1's last
    const long long Pg = ext.P_global > 0 ? ext.P_global : (long long)L.P;
    const bool dir = s.bc_kind == HEAT_BC_DIRICHLET;
    int pin_first = (dir && ext.pe_offset == 0) ? 0 : -1;
    int pin_last = (dir && ext.pe_offset + (long long)L.P == Pg) ? int(L.P) - 1 : -1;
    if (init) {
        std::vector<PeLink> links;
        std::vector<SeedOp> seeds;
        build_links(L, base, s, ext, links, seeds, pin_first, pin_last);
        std::vector<unsigned long long> stats0(kStatWords, 0);
        stats0[kStatLagMin] = ~0ull;
        HB_CUDA(cudaMemcpyAsync(base + L.o_links, links.data(), links.size() * sizeof(PeLink),
                                cudaMemcpyHostToDevice, st));
        HB_CUDA(cudaMemcpyAsync(base + L.o_offL, offL.data(), L.P * 4, cudaMemcpyHostToDevice, st));
        HB_CUDA(cudaMemcpyAsync(base + L.o_offR, offR.data(), L.P * 4, cudaMemcpyHostToDevice, st));
        HB_CUDA(cudaMemcpyAsync(base + L.o_stats, stats0.data(), kStatWords * 8,
                                cudaMemcpyHostToDevice, st));
        HB_TRY(launch_seed(st, bufs[cur], seeds, at<SeedOp>(base, L.o_seeds),
                           2 * L.P + 2 * size_t(L.G)));
    }
    if (steps == 0) return HEAT_OK;
    if (s.mode == 0 && s.law == HEAT_DELAY_GEOMETRIC) {  // exact device delays of the law
        std::vector<uint64_t> gthr;
        HB_TRY(geometric_thresholds(s.geometric_p, s.q, gthr));
        if (!gthr.empty())
            HB_CUDA(cudaMemcpyAsync(base + L.o_gthr, gthr.data(), gthr.size() * sizeof(uint64_t),
                                    cudaMemcpyHostToDevice, st));
    }
    HB_CUDA(cudaMemsetAsync(base + L.o_done, 0, L.P * L.Tp * 4, st));
    HB_CUDA(cudaMemsetAsync(base + L.o_counter, 0, 8, st));
    HB_CUDA(cudaMemsetAsync(base + L.o_abort, 0, 4, st));

    AsyncStreamArgs a{};
    a.buf[0] = bufs[cur];
    a.buf[1] = bufs[cur ^ 1];
    a.N = (long long)s.N;
    a.n = (long long)s.n;
    a.P = int(L.P);
    a.Tp = int(L.Tp);
    a.r = s.r;
    a.c = 1.0 - 2.0 * s.r;  // core.hpp:108
    a.c1 = s.c1;
    a.c2 = s.c2;
    a.dirichlet = s.bc_kind == HEAT_BC_DIRICHLET;
    a.k0 = (long long)k0;
    a.steps = (long long)steps;
    a.s = L.H;  // steps per pass = the halo
    a.npass = (a.steps + a.s - 1) / a.s;
    a.mode = s.mode;
    a.q = int(s.q);
    a.R = L.R;
    a.law = s.law;
    a.fixed_d = int(std::min<size_t>(s.fixed_d, 1u << 30));
    a.seed = s.seed;
    a.modq = make_modq(unsigned(s.q));
    a.D = L.D;
    a.off_left = at<const int>(base, L.o_offL);
    a.off_right = at<const int>(base, L.o_offR);
    a.gthr = at<const uint64_t>(base, L.o_gthr);
    a.links = at<const PeLink>(base, L.o_links);
    a.pin_first_pe = pin_first;
    a.pin_last_pe = pin_last;
    a.done = at<unsigned int>(base, L.o_done);
    a.counter = at<unsigned long long>(base, L.o_counter);
    a.stats = at<unsigned long long>(base, L.o_stats);
    a.flag = flag;
    a.abort_word = at<unsigned int>(base, L.o_abort);
    a.timeout_ns = 20ull * 1000 * 1000 * 1000;
    a.pend_max = stream_pend_max();
    a.edge_log = logs ? logs->edge_log : nullptr;
    a.used_log = logs ? logs->used_log : nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (device_ms) {
        HB_CUDA(cudaEventCreate(&e0));
        HB_CUDA(cudaEventCreate(&e1));
        HB_CUDA(cudaEventRecord(e0, st));
    }
    if (L.V == 32)
        HB_TRY((launch_stream<32, 32>(sms, st, bufs, cur, (long long)s.N, a)));
    else if (L.H == 32)
        HB_TRY((launch_stream<48, 32>(sms, st, bufs, cur, (long long)s.N, a)));
    else
        HB_TRY((launch_stream<48, 64>(sms, st, bufs, cur, (long long)s.N, a)));
    if (device_ms) {
        HB_CUDA(cudaEventRecord(e1, st));
        HB_CUDA(cudaEventSynchronize(e1));
        HB_CUDA(cudaEventElapsedTime(device_ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    if (a.npass & 1) cur ^= 1;
    return HEAT_OK;
}

int async_stream_run(DevCtx& d, const AsyncRunSpec& s, double* bufs[2], int& cur, size_t stride,
                     const std::function<int(size_t, const double*)>& on_record,
                     unsigned long long* host_stats, float* device_ms, const StreamLogs* logs) {
    StreamLayout L;
    std::vector<int> offL, offR;
    const StreamExternal ext{};
    HB_TRY(stream_layout(s, virtual_device_groups(s.N / s.n), ext, L, offL, offR));
    HB_TRY(ensure_scratch(d, L.bytes));
    char* base = static_cast<char*>(d.scratch);
    cudaStream_t st = d.stream;
    HB_CUDA(cudaMemsetAsync(d.flag, 0, 2 * sizeof(unsigned int), st));
    HB_TRY(async_stream_advance(d.sms, st, bufs, cur, s, L, base, ext, offL, offR, 0, 0, true,
                                d.flag, nullptr));
    float total_ms = 0.f;
    size_t k = 0;
    while (k < s.k_end) {
        const size_t next = stride ? std::min(s.k_end, (k / stride + 1) * stride) : s.k_end;
        float ms = 0.f;
        HB_TRY(async_stream_advance(d.sms, st, bufs, cur, s, L, base, ext, offL, offR, k, next - k,
                                    false, d.flag, device_ms ? &ms : nullptr, logs));
        total_ms += ms;
        k = next;
        unsigned int flags[2] = {0, 0};
        HB_CUDA(cudaMemcpyAsync(flags, d.flag, sizeof flags, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
        if (flags[1]) return fail(HEAT_ETIMEOUT, "async halo-ring wait exceeded its deadline");
        if (flags[0]) {
            if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by async step");
            return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
        }
        if (stride && on_record) HB_TRY(on_record(k, bufs[cur]));
    }
    if (device_ms) *device_ms = total_ms;
    if (host_stats)
        HB_CUDA(cudaMemcpy(host_stats, base + L.o_stats, kStatWords * 8, cudaMemcpyDeviceToHost));
    return HEAT_OK;
}

}  // namespace hb

extern "C" int heat_k5_geometry(size_t n, int* points_per_lane, int* halo) {
    return hb::heat_k5_geometry_query(n, points_per_lane, halo);
}

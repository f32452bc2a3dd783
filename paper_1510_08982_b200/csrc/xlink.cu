// xlink.cu -- multi-GPU slabs of the asynchronous (and, with q = 1, exactly
// synchronous) FTCS run: halos travel as P2P stores over NVLink, NCCL only
// carries the 64-byte IPC handles at setup (north star (3)).
//
// Each rank r owns n_local consecutive points split into PEs.  Its K5
// scratch holds two RECEIVE rings: values of the left rank's last point and
// of the right rank's first point.  The neighbours' boundary tiles write
// those rings with st.relaxed.sys + st.release.sys on the progress word;
// this rank's boundary tiles read them locally with ld.acquire.sys.  Nothing
// on the data path goes through the host or a collective, and no rank ever
// waits for more than its two neighbours.
#include <cstring>
#include <memory>

#include "stream_host.cuh"

struct heat_xlink {
    size_t per_pe = 0, q = 0;
    int bc_kind = 0;
    hb::AsyncRunSpec spec{};
    hb::StreamLayout L{};
    hb::StreamExternal ext{};
    std::vector<int> offL, offR;
    void* opened[2] = {nullptr, nullptr};  // IPC mappings to close
};

using namespace hb;

extern "C" {

size_t heat_xlink_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

int heat_plan_xlink_setup(heat_plan* p, size_t per_pe, size_t q, int bc_kind, void* handle_out) {
    if (!p || !handle_out) return fail(HEAT_EINVAL, "null plan or handle buffer");
    if (p->world < 2) return fail(HEAT_EINVAL, "xlink needs a slab plan of a world >= 2");
    if (per_pe == 0 || p->n % per_pe != 0) return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (per_pe <= 32 * 32) return fail(HEAT_EINVAL, "xlink: PEs must be wider than 1024 points");
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    HB_CUDA(cudaSetDevice(p->device));
    // a second setup replaces the first: close its IPC mappings before the
    // scratch they point into is freed and re-exported
    xlink_release(p);
    std::unique_ptr<heat_xlink> x(new heat_xlink());  // owned until stored in p->xlink
    x->per_pe = per_pe;
    x->q = q;
    x->bc_kind = bc_kind;
    x->spec = AsyncRunSpec{p->n, per_pe, 0.0, bc_kind, 0.0, 0.0, 1, q, HEAT_DELAY_UNIFORM,
                           0, 0.5, 0, 0, false};
    const long long P = (long long)(p->n / per_pe);
    x->ext.pe_offset = (long long)p->rank * P;
    x->ext.P_global = (long long)p->world * P;
    const bool periodic = bc_kind == HEAT_BC_PERIODIC;
    x->ext.left = p->rank > 0 || periodic;
    x->ext.right = p->rank + 1 < p->world || periodic;
    HB_TRY(stream_layout(x->spec, 1, x->ext, x->L, x->offL, x->offR));
    // the whole K5 scratch is one IPC-exportable allocation; peers address
    // its receive rings at the layout's offsets (identical on every rank)
    if (p->async_scratch) cudaFree(p->async_scratch);
    p->async_scratch = nullptr;
    p->async_bytes = 0;
    HB_CUDA(cudaMalloc(&p->async_scratch, x->L.bytes));
    HB_CUDA(cudaMemset(p->async_scratch, 0, x->L.bytes));
    // cudaMemset may return before it runs: the zeroing must be done before the
    // handle leaves this process, or it could land after a neighbour's seed
    // stores into our receive rings (seen once with 3 ranks sharing one GPU)
    HB_CUDA(cudaDeviceSynchronize());
    p->async_bytes = x->L.bytes;
    cudaIpcMemHandle_t h;
    HB_CUDA(cudaIpcGetMemHandle(&h, p->async_scratch));
    std::memcpy(handle_out, &h, sizeof h);
    p->xlink = x.release();
    return HEAT_OK;
}

int heat_plan_xlink_connect(heat_plan* p, const void* left_handle, const void* right_handle) {
    if (!p || !p->xlink) return fail(HEAT_EINVAL, "xlink not set up");
    heat_xlink* x = static_cast<heat_xlink*>(p->xlink);
    if (x->ext.left != (left_handle != nullptr) || x->ext.right != (right_handle != nullptr))
        return fail(HEAT_EINVAL, "xlink: neighbour handles do not match the slab's position");
    HB_CUDA(cudaSetDevice(p->device));
    void* lb = nullptr;
    void* rb = nullptr;
    if (left_handle) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, left_handle, sizeof h);
        HB_CUDA(cudaIpcOpenMemHandle(&lb, h, cudaIpcMemLazyEnablePeerAccess));
        x->opened[0] = lb;
    }
    if (right_handle) {
        if (left_handle && std::memcmp(left_handle, right_handle, sizeof(cudaIpcMemHandle_t)) == 0) {
            rb = lb;  // 2-rank periodic ring: the same peer on both sides
        } else {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, right_handle, sizeof h);
            HB_CUDA(cudaIpcOpenMemHandle(&rb, h, cudaIpcMemLazyEnablePeerAccess));
            x->opened[1] = rb;
        }
    }
    // my first point -> the left rank's receive ring for ITS right neighbour;
    // my last point  -> the right rank's receive ring for ITS left neighbour
    if (lb) {
        x->ext.left_push_ring = reinterpret_cast<double*>(static_cast<char*>(lb) + x->L.o_recvR);
        x->ext.left_push_prog =
            reinterpret_cast<unsigned long long*>(static_cast<char*>(lb) + x->L.o_rprogR);
    }
    if (rb) {
        x->ext.right_push_ring = reinterpret_cast<double*>(static_cast<char*>(rb) + x->L.o_recvL);
        x->ext.right_push_prog =
            reinterpret_cast<unsigned long long*>(static_cast<char*>(rb) + x->L.o_rprogL);
    }
    return HEAT_OK;
}

int heat_plan_xlink_seed(heat_plan* p) {
    if (!p || !p->xlink) return fail(HEAT_EINVAL, "xlink not set up");
    heat_xlink* x = static_cast<heat_xlink*>(p->xlink);
    HB_CUDA(cudaSetDevice(p->device));
    return stream_seed_external(p->stream, p->bufs[p->cur], x->spec, x->ext);
}

int heat_plan_xlink_advance(heat_plan* p, double r, double c1, double c2, int mode, int law,
                            size_t fixed_delay, double geometric_p, uint64_t seed, size_t steps,
                            heat_async_stats* stats) {
    if (!p || !p->xlink) return fail(HEAT_EINVAL, "xlink not set up");
    heat_xlink* x = static_cast<heat_xlink*>(p->xlink);
    if (mode != 0 && mode != 1) return fail(HEAT_EINVAL, "xlink: mode is 0 (replay) or 1 (free)");
    if (law == HEAT_DELAY_GEOMETRIC && (!(geometric_p > 0.0) || geometric_p > 1.0))
        return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
    if (law == HEAT_DELAY_FIXED && fixed_delay >= x->q)
        return fail(HEAT_EDOMAIN, "DelayModel: fixed delay must satisfy d < q");
    HB_CUDA(cudaSetDevice(p->device));
    AsyncRunSpec s = x->spec;
    s.r = r;
    s.c1 = c1;
    s.c2 = c2;
    s.mode = mode;
    s.law = law;
    s.fixed_d = fixed_delay;
    s.geometric_p = geometric_p;
    s.seed = seed;
    s.k_end = steps;
    char* base = static_cast<char*>(p->async_scratch);
    // local rings + links (the receive rings were seeded by the neighbours;
    // the caller barriers between heat_plan_xlink_seed and this call)
    HB_TRY(async_stream_advance(p->sms, p->stream, p->bufs, p->cur, s, x->L, base, x->ext, x->offL,
                                x->offR, 0, 0, true, p->flag, nullptr));
    HB_TRY(async_stream_advance(p->sms, p->stream, p->bufs, p->cur, s, x->L, base, x->ext, x->offL,
                                x->offR, 0, steps, false, p->flag, nullptr));
    if (stats) {
        std::vector<unsigned long long> hs(kStatWords, 0);
        HB_CUDA(cudaMemcpyAsync(hs.data(), base + x->L.o_stats, kStatWords * 8,
                                cudaMemcpyDeviceToHost, p->stream));
        HB_CUDA(cudaStreamSynchronize(p->stream));
        std::memset(stats, 0, sizeof *stats);
        stats->reads = hs[kStatReads];
        stats->waits = hs[kStatWaits];
        stats->max_delay = hs[kStatMaxDelay];
        for (int i = 0; i < 64; ++i) stats->delay_histogram[i] = hs[kStatDelayHist + i];
    }
    return HEAT_OK;
}

int heat_plan_xlink_debug_recv(heat_plan* p, double* out2) {
    if (!p || !p->xlink || !out2) return fail(HEAT_EINVAL, "xlink not set up");
    heat_xlink* x = static_cast<heat_xlink*>(p->xlink);
    HB_CUDA(cudaSetDevice(p->device));
    HB_CUDA(cudaStreamSynchronize(p->stream));
    char* base = static_cast<char*>(p->async_scratch);
    HB_CUDA(cudaMemcpy(&out2[0], base + x->L.o_recvL, sizeof(double), cudaMemcpyDeviceToHost));
    HB_CUDA(cudaMemcpy(&out2[1], base + x->L.o_recvR, sizeof(double), cudaMemcpyDeviceToHost));
    return HEAT_OK;
}

}  // extern "C"

namespace hb {
void xlink_release(heat_plan* p) {
    if (!p->xlink) return;
    heat_xlink* x = static_cast<heat_xlink*>(p->xlink);
    for (void* o : x->opened)
        if (o) cudaIpcCloseMemHandle(o);
    delete x;
    p->xlink = nullptr;
}
}  // namespace hb

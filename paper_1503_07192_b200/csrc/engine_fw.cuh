// engine_fw.cuh — contexts and the blocked Floyd-Warshall drivers (1 GPU and row-sharded over NCCL), value-kind selection.
// Internal to libpsp_gpu.so (one translation unit: psp_gpu.cu includes the
// engine headers in dependency order).
#pragma once

// --------------------------------------------------------------- ctx ----
struct psp_gpu_ctx {
    int device = 0;
    int rank = 0, world = 1;
    int sms = 148;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;  // world > 1 only
    int storage = PSP_STORAGE_REPLICATED;  // boundary-graph table of later builds
};

namespace {

int g_attr_done[2] = {0, 0};
template <class V> constexpr int P3_SMEM = 3 * TT * sizeof(V);  // A + 2 x B

template <class V>
void set_kernel_attrs() {
    const int idx = std::is_same<V, float>::value ? 1 : 0;
    if (g_attr_done[idx]) return;
    const int smem = 2 * TT * sizeof(V);
    CK(cudaFuncSetAttribute(fw_phase2<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(fw_phase3<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, P3_SMEM<V>));
    g_attr_done[idx] = 1;
}

template <class V>
void fill_arena(MatArena& a, cudaStream_t s, int sms) {
    for (const auto& r : a.backed_ranges()) {  // all of it unless row-sharded
        const uint64_t n = r.second / sizeof(V);
        const int blocks = int(std::min<uint64_t>((n + 255) / 256, uint64_t(sms) * 32));
        fill_value<V><<<std::max(blocks, 1), 256, 0, s>>>(a.tiles_as<V>() + r.first / sizeof(V), n,
                                                          Ops<V>::inf());
        CK_LAUNCH();
    }
    if (a.nmat) {
        set_diag_zero<V><<<a.nmat, 256, 0, s>>>(a.view<V>());
        CK_LAUNCH();
    }
}

void read_walked_tiles(MatArena& a, cudaStream_t s) {
    unsigned long long t = 0;
    CK(cudaMemcpyAsync(&t, a.act_work_ptr(), sizeof(t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    a.walked_tiles = t;
}

#define NCK(x)                                                                         \
    do {                                                                               \
        ncclResult_t r_ = (x);                                                         \
        if (r_ != ncclSuccess)                                                         \
            throw Fail{PSP_ENCCL, std::string(#x) + ": " + nccl().GetErrorString(r_)}; \
    } while (0)

template <class V> ncclDataType_t nccl_type();
template <> ncclDataType_t nccl_type<uint32_t>() { return ncclUint32; }
template <> ncclDataType_t nccl_type<float>() { return ncclFloat32; }

// Sparse walk: per-matrix active lists, then the prefix over matrices.
template <class V>
void launch_active_list(const MatSet<V>& v, uint32_t kb, cudaStream_t s) {
    fw_active_list<V><<<v.nmat, 1024, 0, s>>>(v, kb);
    CK_LAUNCH();
    fw_mat_prefix<V><<<1, 1024, 0, s>>>(v);
    CK_LAUNCH();
}

// The blocked FW driver over a set of matrices: 3 launches per k-block on
// one stream (5 with the sparse walk's work lists).
template <class V>
void run_fw_set(const MatSet<V>& v, uint32_t nb_max, uint64_t work, cudaStream_t s, int sms) {
    if (v.nmat == 0 || nb_max == 0) return;
    set_kernel_attrs<V>();
    const int smem = 2 * TT * sizeof(V);
    const int g3 = int(std::max<uint64_t>(1, std::min<uint64_t>(work, uint64_t(sms))));
    if (v.act_flag) CK(cudaMemsetAsync(v.act_work, 0, sizeof(unsigned long long), s));
    // PSP_K2_TRACE=file: per k-block active slots and phase-3 tiles of a
    // single sparse matrix (diagnostic; synchronises every k-block)
    const char* trace = v.nmat == 1 && v.act_flag ? std::getenv("PSP_K2_TRACE") : nullptr;
    FILE* tf = trace ? std::fopen(trace, "w") : nullptr;
    for (uint32_t kb = 0; kb < nb_max; ++kb) {
        fw_phase1<V><<<v.nmat, NTHREADS, 0, s>>>(v, kb);
        CK_LAUNCH();
        if (nb_max > 1) {
            fw_phase2<V><<<dim3(v.nmat, nb_max), NTHREADS, smem, s>>>(v, kb);
            CK_LAUNCH();
            if (v.act_flag) launch_active_list<V>(v, kb, s);
            if (tf) {
                uint32_t meta[2];
                uint64_t tot = 0;
                CK(cudaMemcpyAsync(meta, v.act_meta, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaMemcpyAsync(&tot, v.mat_prefix + 1, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                std::fprintf(tf, "%u %u %llu\n", kb, meta[0], (unsigned long long)tot);
            }
            fw_phase3<V><<<g3, NTHREADS, P3_SMEM<V>, s>>>(v, kb);
            CK_LAUNCH();
        }
    }
    if (tf) std::fclose(tf);
}

template <class V>
void run_fw(const MatArena& a, cudaStream_t s, int sms) {
    if (a.nmat == 0 || a.nb_max == 0) return;
    const MatSet<V> v = a.view<V>();
    run_fw_set<V>(v, a.nb_max, a.work_prefix[a.nmat], s, sms);
    if (v.act_flag) read_walked_tiles(const_cast<MatArena&>(a), s);
}

// Component-sharded K1 (multi-GPU): the k component matrices are
// independent, so rank r closes a contiguous range of them, balanced by FW
// work (ntiles_upper(nb) * nb tiles per matrix), and the ranges are then
// broadcast from their owners, so every GPU ends with the full arena (queries
// stay replicated). Each range is one contiguous run of the tile arena.
inline std::vector<uint32_t> k1_ranges(const MatArena& a, int world) {
    std::vector<uint64_t> cost(a.nmat + 1, 0);
    for (uint32_t m = 0; m < a.nmat; ++m) cost[m + 1] = cost[m] + ntiles_upper(a.nb[m]) * a.nb[m];
    std::vector<uint32_t> cut(world + 1, a.nmat);
    cut[0] = 0;
    uint32_t m = 0;
    for (int r = 1; r < world; ++r) {
        const double goal = double(cost[a.nmat]) * r / world;
        while (m < a.nmat && double(cost[m + 1]) <= goal) ++m;
        cut[r] = std::max(m, cut[r - 1]);
    }
    return cut;
}

// Every rank's range of the component arena from its owner (component-
// sharded K1, see k1_ranges).
template <class V>
void broadcast_component_ranges(const MatArena& a, const std::vector<uint32_t>& cut, psp_gpu_ctx* ctx) {
    const ncclDataType_t dt = nccl_type<V>();
    V* tiles = a.tiles.as<V>();
    NCK(nccl().GroupStart());
    for (int r = 0; r < ctx->world; ++r) {
        const uint64_t e0 = cut[r] < a.nmat ? a.tile_base[cut[r]] : a.tile_elems;
        const uint64_t e1 = cut[r + 1] < a.nmat ? a.tile_base[cut[r + 1]] : a.tile_elems;
        if (e1 > e0) NCK(nccl().Broadcast(tiles + e0, tiles + e0, e1 - e0, dt, r, ctx->comm, ctx->stream));
    }
    NCK(nccl().GroupEnd());
}

template <class V>
void run_fw_components_sharded(const MatArena& a, psp_gpu_ctx* ctx) {
    if (a.nmat == 0 || a.nb_max == 0) return;
    cudaStream_t s = ctx->stream;
    const std::vector<uint32_t> cut = k1_ranges(a, ctx->world);
    const uint32_t m0 = cut[ctx->rank], m1 = cut[ctx->rank + 1];
    if (m1 > m0) {
        // a view of matrices [m0, m1): their own index arrays (work prefix
        // rebased to 0) over the shared tile and panel buffers
        std::vector<uint64_t> tb(a.tile_base.begin() + m0, a.tile_base.begin() + m1);
        std::vector<uint64_t> pb(a.panel_base.begin() + m0, a.panel_base.begin() + m1);
        std::vector<uint32_t> nbv(a.nb.begin() + m0, a.nb.begin() + m1);
        std::vector<uint64_t> wp(m1 - m0 + 1);
        for (uint32_t m = m0; m <= m1; ++m) wp[m - m0] = a.work_prefix[m] - a.work_prefix[m0];
        DBuf d_tb = upload(tb, s), d_pb = upload(pb, s), d_nb = upload(nbv, s), d_wp = upload(wp, s);
        MatSet<V> v = a.view<V>();
        v.tile_base = d_tb.as<uint64_t>();
        v.panel_base = d_pb.as<uint64_t>();
        v.nb = d_nb.as<uint32_t>();
        v.work_prefix = d_wp.as<uint64_t>();
        v.nmat = m1 - m0;
        v.nb_max = *std::max_element(nbv.begin(), nbv.end());
        v.rows = nullptr;
        v.row_prefix = nullptr;
        v.nrows = 0;
        v.rank = 0;
        v.world = 1;
        v.act_flag = nullptr;
        run_fw_set<V>(v, v.nb_max, wp.back(), s, ctx->sms);
        CK(cudaStreamSynchronize(s));  // the index arrays die here
    }
    broadcast_component_ranges<V>(a, cut, ctx);
}


// ------------------------------------------ peer-to-peer panel exchange --
// Every rank of the row-sharded K2 owns an exchange region that all peers map
// (CUDA IPC over NVLink):
//   panel[2][nb][T*T] | flag[2][nb] | diag[2][T*T]  (V, double-buffered by
//   k-block parity) | sync[8] (u64: [0] k-blocks whose diagonal tile this
//   rank published, [1] k-blocks whose panel slots it finished, [7] error)
// Per k-block kb (owner o = kb mod world):
//   o:      phase 1, publish diag[kb&1], sync[0] = kb + 1
//   others: pull_diag - wait for o's sync[0] > kb, copy o's diag into the
//           local tile (kb, kb)
//   all:    phase 2 on the slots this rank owns (home row mod world), into
//           its own panel[kb&1] + flag[kb&1]; sync[1] = kb + 1
//   all:    pull_panel - per slot J owned elsewhere: wait for the owner's
//           sync[1] > kb, copy its activity flag and, only if the slot is
//           active (holds a finite entry), its 64 KB tile
// so the panel moves once per consumer and only where it carries work (the
// NCCL path min-allreduced every slot, active or not). Reuse of a parity
// buffer at kb + 2 is safe: a rank reaches it only after every peer's
// sync[1] passed kb + 1, i.e. after their pulls of kb. Waits time out after
// 60 s (sync[7] = 1, reported as PSP_ECUDA) instead of hanging the GPU.
struct P2PRegion {
    size_t panel_off[2], flag_off[2], diag_off[2], sync_off, bytes;
    P2PRegion(uint32_t nb, size_t vb) {
        size_t at = 0;
        auto take = [&](size_t b) {
            const size_t o = at;
            at += (b + 255) / 256 * 256;
            return o;
        };
        for (int i = 0; i < 2; ++i) panel_off[i] = take(size_t(nb) * TT * vb);
        for (int i = 0; i < 2; ++i) flag_off[i] = take(size_t(nb) * vb);
        for (int i = 0; i < 2; ++i) diag_off[i] = take(TT * vb);
        sync_off = take(8 * sizeof(unsigned long long));
        bytes = at;
    }
};

__device__ __forceinline__ unsigned long long fw_global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// wait until *f >= want (a peer's counter, read over NVLink); false on timeout
__device__ bool wait_counter(const volatile unsigned long long* f, unsigned long long want,
                             volatile unsigned long long* err) {
    const unsigned long long t0 = fw_global_ns();
    while (*f < want) {
        if (*err) return false;
        if (fw_global_ns() - t0 > 60ull * 1000 * 1000 * 1000) {
            *err = 1;
            return false;
        }
        __nanosleep(64);
    }
    return true;
}

__global__ void p2p_signal(unsigned long long* f, unsigned long long v) {
    // the previous kernels of this stream are complete: their writes are in
    // this GPU's memory, where the peers' NVLink loads are served
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(f) = v;
    __threadfence_system();
}

// copy the owner's published diagonal tile (TT values) into the local tile
template <class V>
__global__ void __launch_bounds__(256) pull_diag(const V* src, const unsigned long long* src_sync,
                                                 unsigned long long want, V* dst,
                                                 unsigned long long* err) {
    __shared__ int ok;
    if (threadIdx.x == 0)
        ok = wait_counter(reinterpret_cast<const volatile unsigned long long*>(src_sync), want,
                          reinterpret_cast<volatile unsigned long long*>(err));
    __syncthreads();
    if (!ok) return;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    constexpr uint32_t n4 = TT * sizeof(V) / 16;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
        d4[i] = s4[i];
}

// one CTA per panel slot J != kb owned by another rank: its flag, and its
// tile when active, from the owner's region into this rank's
template <class V>
__global__ void __launch_bounds__(256) pull_panel(unsigned char* const* peers, P2PRegion lay,
                                                  int buf, uint32_t kb, uint32_t nb, uint32_t rank,
                                                  uint32_t world, V* panel, V* flag,
                                                  unsigned long long* err) {
    const uint32_t J = blockIdx.x;
    if (J == kb) return;
    const uint32_t o = (J > kb ? kb : J) % world;  // home row's owner
    if (o == rank) return;
    const unsigned char* peer = peers[o];
    __shared__ int act;
    if (threadIdx.x == 0) {
        act = 0;
        if (wait_counter(reinterpret_cast<const volatile unsigned long long*>(peer + lay.sync_off) + 1,
                         kb + 1, reinterpret_cast<volatile unsigned long long*>(err))) {
            const V f = reinterpret_cast<const volatile V*>(peer + lay.flag_off[buf])[J];
            flag[J] = f;
            act = f == V(0);
        }
    }
    __syncthreads();
    if (!act) return;
    const uint4* s4 = reinterpret_cast<const uint4*>(peer + lay.panel_off[buf]) + size_t(J) * (TT * sizeof(V) / 16);
    uint4* d4 = reinterpret_cast<uint4*>(panel) + size_t(J) * (TT * sizeof(V) / 16);
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < TT * sizeof(V) / 16; i += blockDim.x) d4[i] = s4[i];
}

// The exchange regions of all ranks of a sharded build, mapped into this
// process (the peers' through CUDA IPC).
struct P2PExchange {
    P2PRegion lay;
    DBuf region, d_peers;
    std::vector<unsigned char*> base;
    std::vector<void*> opened;
    P2PExchange(uint32_t nb, size_t vb) : lay(nb, vb) {}
    ~P2PExchange() { close_peers(); }
    void close_peers() {
        for (void* p : opened) cudaIpcCloseMemHandle(p);
        opened.clear();
    }
    unsigned char* mine(int rank) const { return base[rank]; }
};

// Sets the exchange up (allocation, zeroed counters, IPC handles gathered
// over NCCL and opened); returns false when the peers cannot be mapped.
template <class V>
bool p2p_setup(P2PExchange& x, psp_gpu_ctx* ctx) {
    cudaStream_t s = ctx->stream;
    const int G = ctx->world;
    x.region.alloc_ipc(x.lay.bytes);
    CK(cudaMemsetAsync(x.region.p, 0, x.lay.bytes, s));
    cudaIpcMemHandle_t mine;
    int ok = cudaIpcGetMemHandle(&mine, x.region.p) == cudaSuccess;
    cudaGetLastError();
    // every rank must agree before anyone uses the path
    {
        uint64_t v = ok;
        DBuf d(8);
        CK(cudaMemcpyAsync(d.p, &v, 8, cudaMemcpyHostToDevice, s));
        NCK(nccl().AllReduce(d.p, d.p, 1, ncclUint64, ncclMin, ctx->comm, s));
        CK(cudaMemcpyAsync(&v, d.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (!v) return false;
    }
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    DBuf dh(hb * G);
    CK(cudaMemcpyAsync(static_cast<char*>(dh.p) + hb * ctx->rank, &mine, hb, cudaMemcpyHostToDevice, s));
    NCK(nccl().AllGather(static_cast<char*>(dh.p) + hb * ctx->rank, dh.p, hb, ncclChar, ctx->comm, s));
    std::vector<cudaIpcMemHandle_t> h(G);
    CK(cudaMemcpyAsync(h.data(), dh.p, hb * G, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    x.base.assign(G, nullptr);
    uint64_t opened_ok = 1;
    for (int r = 0; r < G; ++r) {
        if (r == ctx->rank) {
            x.base[r] = x.region.as<unsigned char>();
            continue;
        }
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, h[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            opened_ok = 0;
            continue;
        }
        x.opened.push_back(p);
        x.base[r] = static_cast<unsigned char*>(p);
    }
    {
        DBuf d(8);
        CK(cudaMemcpyAsync(d.p, &opened_ok, 8, cudaMemcpyHostToDevice, s));
        NCK(nccl().AllReduce(d.p, d.p, 1, ncclUint64, ncclMin, ctx->comm, s));
        CK(cudaMemcpyAsync(&opened_ok, d.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    if (!opened_ok) return false;
    x.d_peers = upload(x.base, s);  // the zeroed counters are in place on every rank (stream order
                                    // + the AllReduce above): peers may signal from here on
    return true;
}

// Row-sharded blocked FW of the boundary graph over ctx->world GPUs
// (SURVEY §8e): tile row I is owned by rank I mod world. Per k-block the
// owner closes the diagonal tile and broadcasts it; every rank updates the
// panel tiles whose home row it owns (others contribute INF) and one
// min-allreduce assembles the full row panel; phase 3 then touches owned rows
// only. At the end every row is broadcast from its owner so each GPU holds
// the complete table (queries stay replicated, no per-query traffic) --
// unless the arena is row-sharded storage (MatArena::part: only the owned
// rows exist on this rank), which stays distributed for routed queries; the
// diagonal tile of a k-block this rank does not own then goes to a scratch
// tile (MatSet::diag) instead of its slot in the table.
template <class V>
void run_fw_sharded(MatArena& a, psp_gpu_ctx* ctx) {
    cudaStream_t s = ctx->stream;
    const uint32_t nb = a.nb[0];
    set_kernel_attrs<V>();
    a.shard_rows(ctx->rank, ctx->world, s);
    const MatSet<V> v = a.view<V>();
    const int smem = 2 * TT * sizeof(V);
    const uint64_t my_work = std::max<uint64_t>(1, a.nrows ? (a.nrows * uint64_t(nb)) : 1);
    const int g3 = int(std::min<uint64_t>(my_work, uint64_t(ctx->sms)));
    const ncclDataType_t dt = nccl_type<V>();
    V* tiles = a.tiles_as<V>();
    const bool row_storage = a.part != nullptr;
    DBuf diag_scratch;
    if (row_storage) diag_scratch.alloc(TT * sizeof(V));
    // PSP_FW_PROFILE=1: per-phase CUDA-event breakdown on stderr (diagnostics)
    const bool prof = std::getenv("PSP_FW_PROFILE") != nullptr;
    const char* dm = std::getenv("PSP_DIAG_MODE");
    const bool diag_allreduce = dm && std::strcmp(dm, "allreduce") == 0;
    cudaEvent_t ev[5];
    double acc_ms[4] = {0, 0, 0, 0};
    if (prof)
        for (auto& e : ev) CK(cudaEventCreate(&e));
    if (v.act_flag) CK(cudaMemsetAsync(v.act_work, 0, sizeof(unsigned long long), s));
    // panel exchange: peer-to-peer pulls of the active slots over NVLink
    // (default with the sparse walk), or PSP_K2_EXCHANGE=nccl: the
    // min-allreduce of every slot
    const char* xenv = std::getenv("PSP_K2_EXCHANGE");
    std::unique_ptr<P2PExchange> x;
    if (v.act_flag && nb > 1 && !(xenv && std::strcmp(xenv, "nccl") == 0)) {
        x = std::make_unique<P2PExchange>(nb, sizeof(V));
        if (!p2p_setup<V>(*x, ctx)) x.reset();  // every rank takes the same branch
    }
    for (uint32_t kb = 0; kb < nb && x; ++kb) {
        const int owner = int(kb % ctx->world);
        const int buf = int(kb & 1);
        V* diag = tiles + tidx(kb, kb, nb) * TT;
        const P2PRegion& L = x->lay;
        unsigned char* me = x->mine(ctx->rank);
        auto* my_sync = reinterpret_cast<unsigned long long*>(me + L.sync_off);
        MatSet<V> vk = v;
        vk.p2p = 1;
        vk.panel = reinterpret_cast<V*>(me + L.panel_off[buf]);
        vk.act_flag = reinterpret_cast<V*>(me + L.flag_off[buf]);
        if (prof) CK(cudaEventRecord(ev[0], s));
        if (owner == ctx->rank) {
            fw_phase1<V><<<1, NTHREADS, 0, s>>>(vk, kb);
            CK_LAUNCH();
            CK(cudaMemcpyAsync(me + L.diag_off[buf], diag, TT * sizeof(V), cudaMemcpyDeviceToDevice, s));
            p2p_signal<<<1, 1, 0, s>>>(my_sync, kb + 1);
            CK_LAUNCH();
        } else {
            const unsigned char* ob = x->base[owner];
            V* dst = diag;
            if (row_storage) vk.diag = dst = diag_scratch.as<V>();
            pull_diag<V><<<16, 256, 0, s>>>(reinterpret_cast<const V*>(ob + L.diag_off[buf]),
                                            reinterpret_cast<const unsigned long long*>(ob + L.sync_off),
                                            kb + 1, dst, my_sync + 7);
            CK_LAUNCH();
        }
        if (prof) CK(cudaEventRecord(ev[1], s));
        fw_phase2<V><<<dim3(1, nb), NTHREADS, smem, s>>>(vk, kb);
        CK_LAUNCH();
        p2p_signal<<<1, 1, 0, s>>>(my_sync + 1, kb + 1);
        CK_LAUNCH();
        if (prof) CK(cudaEventRecord(ev[2], s));
        pull_panel<V><<<nb, 256, 0, s>>>(x->d_peers.as<unsigned char*>(), L, buf, kb, nb,
                                         uint32_t(ctx->rank), uint32_t(ctx->world), vk.panel,
                                         vk.act_flag, my_sync + 7);
        CK_LAUNCH();
        if (prof) CK(cudaEventRecord(ev[3], s));
        launch_active_list<V>(vk, kb, s);
        fw_phase3<V><<<ctx->sms, NTHREADS, P3_SMEM<V>, s>>>(vk, kb);
        CK_LAUNCH();
        if (prof) {
            CK(cudaEventRecord(ev[4], s));
            CK(cudaEventSynchronize(ev[4]));
            for (int i = 0; i < 4; ++i) {
                float t = 0;
                CK(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
                acc_ms[i] += t;
            }
        }
    }
    if (x) {
        unsigned long long err = 0;
        CK(cudaMemcpyAsync(&err, x->mine(ctx->rank) + x->lay.sync_off + 7 * sizeof(err), sizeof(err),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (err) throw Fail{PSP_ECUDA, "K2 panel exchange: a peer did not signal within 60 s"};
    }
    for (uint32_t kb = 0; kb < nb && !x; ++kb) {
        const int owner = int(kb % ctx->world);
        V* diag = tiles + tidx(kb, kb, nb) * TT;
        if (prof) CK(cudaEventRecord(ev[0], s));
        if (owner == ctx->rank) {
            fw_phase1<V><<<1, NTHREADS, 0, s>>>(v, kb);
            CK_LAUNCH();
        }
        MatSet<V> vk = v;
        if (row_storage && owner != ctx->rank) {
            vk.diag = diag_scratch.as<V>();
            NCK(nccl().Broadcast(diag, diag_scratch.p, TT, dt, owner, ctx->comm, s));
        } else if (diag_allreduce) {
            // owners contribute the closed tile, everyone else INF
            if (owner != ctx->rank) fill_value<V><<<16, 256, 0, s>>>(diag, TT, Ops<V>::inf());
            NCK(nccl().AllReduce(diag, diag, TT, dt, ncclMin, ctx->comm, s));
        } else {
            NCK(nccl().Broadcast(diag, diag, TT, dt, owner, ctx->comm, s));
        }
        if (prof) CK(cudaEventRecord(ev[1], s));
        if (nb > 1) {
            fw_phase2<V><<<dim3(1, nb), NTHREADS, smem, s>>>(vk, kb);
            CK_LAUNCH();
            if (prof) CK(cudaEventRecord(ev[2], s));
            // sparse: the activity flags follow the panel slots in the same buffer
            NCK(nccl().AllReduce(a.panel.p, a.panel.p, uint64_t(nb) * TT + (v.act_flag ? nb : 0), dt,
                                 ncclMin, ctx->comm, s));
            if (prof) CK(cudaEventRecord(ev[3], s));
            if (v.act_flag) {
                launch_active_list<V>(v, kb, s);
                fw_phase3<V><<<ctx->sms, NTHREADS, P3_SMEM<V>, s>>>(v, kb);
                CK_LAUNCH();
            } else if (a.nrows) {
                fw_phase3<V><<<g3, NTHREADS, P3_SMEM<V>, s>>>(v, kb);
                CK_LAUNCH();
            }
            if (prof) {
                CK(cudaEventRecord(ev[4], s));
                CK(cudaEventSynchronize(ev[4]));
                for (int i = 0; i < 4; ++i) {
                    float t = 0;
                    CK(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
                    acc_ms[i] += t;
                }
            }
        }
    }
    if (prof) {
        std::fprintf(stderr,
                     "[psp] rank %d sharded FW nb=%u (%s exchange): phase1+diag %.1f ms, phase2 %.1f "
                     "ms, panel exchange %.1f ms, phase3 %.1f ms\n",
                     ctx->rank, nb, x ? "p2p" : "nccl", acc_ms[0], acc_ms[1], acc_ms[2], acc_ms[3]);
        for (auto& e : ev) cudaEventDestroy(e);
    }
    if (v.act_flag) {  // total phase-3 tiles over all ranks
        NCK(nccl().AllReduce(v.act_work, v.act_work, 1, ncclUint64, ncclSum, ctx->comm, s));
        read_walked_tiles(a, s);
    }
    if (x) {
        // no rank may free its region while a peer still maps it: close the
        // imports, then a barrier, then the regions go (CUDA IPC rules)
        CK(cudaStreamSynchronize(s));
        x->close_peers();
        DBuf d(8);
        CK(cudaMemsetAsync(d.p, 0, 8, s));
        NCK(nccl().AllReduce(d.p, d.p, 1, ncclUint64, ncclMax, ctx->comm, s));
        CK(cudaStreamSynchronize(s));
        x.reset();
    }
    if (row_storage) {
        CK(cudaStreamSynchronize(s));  // the diagonal scratch dies here
        return;
    }
    // replicate: row I (tiles (I, I..nb-1), contiguous) from its owner
    const uint32_t batch = 64;
    for (uint32_t I0 = 0; I0 < nb; I0 += batch) {
        NCK(nccl().GroupStart());
        for (uint32_t I = I0; I < std::min(nb, I0 + batch); ++I) {
            V* row = tiles + tidx(I, I, nb) * TT;
            NCK(nccl().Broadcast(row, row, uint64_t(nb - I) * TT, dt, int(I % ctx->world),
                                 ctx->comm, s));
        }
        NCK(nccl().GroupEnd());
    }
}

// Value kind selection: u32 when integral or dyadic weights keep
// every finite distance below INF; f32 otherwise.
struct Kind {
    int kind;
    int shift;
};
Kind choose_kind(int requested, const double* w, uint64_t m, uint64_t n) {
    if (requested != PSP_VALUE_AUTO && requested != PSP_VALUE_U32 && requested != PSP_VALUE_F32)
        throw ArgError("value_kind must be PSP_VALUE_AUTO, PSP_VALUE_U32 or PSP_VALUE_F32");
    if (requested == PSP_VALUE_F32) return {PSP_VALUE_F32, 0};
    double maxw = 0.0;
    for (uint64_t e = 0; e < m; ++e) maxw = std::max(maxw, w[e]);
    const double hops = n > 1 ? double(n - 1) : 1.0;
    for (int q = 0; q <= 24; ++q) {
        const double scale = std::ldexp(1.0, q);
        if (maxw * scale * hops >= double(U32_INF)) break;
        bool integral = true;
        for (uint64_t e = 0; e < m && integral; ++e) {
            const double x = w[e] * scale;
            integral = std::floor(x) == x;
        }
        if (integral) return {PSP_VALUE_U32, q};
    }
    if (requested == PSP_VALUE_U32)
        throw Fail{PSP_EOVERFLOW,
                   "u32 distances are not exact for these weights (non-dyadic weights or "
                   "max_w * 2^q * (n-1) >= 2^31-1)"};
    return {PSP_VALUE_F32, 0};
}

template <class V>
V to_value(double w, int shift) {
    if (std::is_same<V, float>::value) return V(float(w));
    return V(static_cast<uint32_t>(std::ldexp(w, shift)));
}

template <class V>
void to_f64(const std::vector<V>& src, double* dst, double scale) {
    for (size_t i = 0; i < src.size(); ++i) {
        if (std::is_same<V, float>::value) {
            dst[i] = double(src[i]);
        } else {
            const uint32_t v = static_cast<uint32_t>(src[i]);
            dst[i] = v >= U32_INF ? HUGE_VAL : double(v) * scale;
        }
    }
}

}  // namespace


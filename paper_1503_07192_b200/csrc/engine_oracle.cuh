// engine_oracle.cuh — the device oracle: build (K0-K2), import, export, query launchers.
// Internal to libpsp_gpu.so (one translation unit: psp_gpu.cu includes the
// engine headers in dependency order).
#pragma once

// ------------------------------------------------------------ oracle ----
// Grow-only workspace of the grouped query kernel, and the event that
// serialises its reuse across caller streams.
struct GroupWorkspace {
    DBuf buf, bins, temp, tasks;
    uint64_t count = 0;
    size_t temp_bytes = 0;
    cudaEvent_t done = nullptr;
    GroupWorkspace() = default;
    GroupWorkspace(const GroupWorkspace&) = delete;
    GroupWorkspace& operator=(const GroupWorkspace&) = delete;
    ~GroupWorkspace() {
        if (done) cudaEventDestroy(done);
    }
};

struct psp_gpu_oracle {
    psp_gpu_ctx* ctx = nullptr;
    Kind kind{PSP_VALUE_U32, 0};
    double scale = 1.0;
    Reordered R;
    MatArena comps, bg;
    DBuf d_perm, d_assign, d_comp_off, d_bnd_off, d_cb_off, d_cb;
    uint64_t device_bytes = 0;
    // PSP_STORAGE_ROW_SHARDED build (world > 1): `bg` is the K2 working
    // matrix with only this rank's tile rows backed (MatArena::part);
    // boundary id i sits at position d_bg_pos[i] of it. The oracle then
    // answers through psp_gpu_shard (routed queries) only.
    bool row_storage = false;
    DBuf d_bg_pos;
    // grow-only staging for the host-pointer query API (one call at a time;
    // the tables themselves are read-only, src/query.cpp is re-entrant too)
    std::mutex query_mu;
    DBuf query_stage;
    // pinned host staging of small host batches (<= kPinnedPairs pairs):
    // pairs in, bad-id flag + distances out, one DMA each way and one sync.
    // cfg3 e2e: 1K pairs 15.3 -> 22.3 M queries/s; from ~100K pairs the host
    // memcpy into the staging costs more than it saves (1M: 146 -> 132 M)
    static constexpr uint64_t kPinnedPairs = 1u << 14;
    void* host_stage = nullptr;
    size_t host_stage_bytes = 0;
    GroupWorkspace gw;
    // per-stream workspaces for callers on their own streams (concurrent
    // batches then run side by side; beyond kStreamWorkspaces streams they
    // share `gw`, ordered by its event). Guarded by query_mu.
    static constexpr size_t kStreamWorkspaces = 8;
    std::map<cudaStream_t, std::unique_ptr<GroupWorkspace>> stream_gw;
    GroupWorkspace& workspace_for(cudaStream_t s) {
        if (s == ctx->stream) return gw;
        auto it = stream_gw.find(s);
        if (it != stream_gw.end()) return *it->second;
        if (stream_gw.size() >= kStreamWorkspaces) return gw;
        return *stream_gw.emplace(s, std::make_unique<GroupWorkspace>()).first->second;
    }
    // block query layout of the boundary table (optional, see
    // build_query_blocks): BQ blocks and their offsets
    DBuf bq, d_bq_off;
    // 16-bit residual layout (u32 tables, build_query_blocks16)
    DBuf bq16, d_bq16_off, bqaux, d_aux_off, cb16, d_cb16_off, d_rbase;
    uint32_t u16_sat = 0x7FFFu;
    // point-query server (query_server): mailbox in mapped pinned host
    // memory, its stream, the last request number. Guarded by query_mu.
    QueryMailbox* mb = nullptr;
    cudaStream_t srv = nullptr;
    unsigned long long srv_seq = 0;
    // PSP_SERVER_PROFILE: calls, host round trip and device time (ns)
    double srv_prof[3] = {0, 0, 0};
    psp_gpu_oracle() = default;
    psp_gpu_oracle(const psp_gpu_oracle&) = delete;
    psp_gpu_oracle& operator=(const psp_gpu_oracle&) = delete;
    ~psp_gpu_oracle() {
        if (srv_prof[0] > 0)
            std::fprintf(stderr,
                         "[psp] point-query server: %.0f calls, %.3f us host round trip, %.3f us "
                         "on the device (request seen -> answered)\n",
                         srv_prof[0], srv_prof[1] / srv_prof[0] / 1e3, srv_prof[2] / srv_prof[0] / 1e3);
        if (srv) {
            cudaStreamSynchronize(srv);  // the server exits after its idle time
            cudaStreamDestroy(srv);
        }
        if (mb) cudaFreeHost(mb);
        if (host_stage) cudaFreeHost(host_stage);
    }
};

namespace {

// Operations that read the whole boundary-graph table from this GPU.
void require_replicated(const psp_gpu_oracle* o, const char* what) {
    if (o->row_storage)
        throw ArgError(std::string(what) +
                       ": the boundary-graph table is row-sharded over the ranks "
                       "(PSP_STORAGE_ROW_SHARDED); query through psp_gpu_shard_create + "
                       "psp_gpu_routed_query_batch");
}

struct EdgeLists {
    std::vector<uint32_t> mat, ii, jj;  // intra-component (local ids)
    std::vector<double> w;
    std::vector<uint32_t> bi, bj;       // cross edges (boundary ids)
    std::vector<double> bw;
};

EdgeLists split_edges(const Reordered& R) {
    EdgeLists L;
    const Csr& g = R.g;
    for (uint64_t u = 0; u < R.n; ++u) {
        const uint32_t cu = R.assign[u];
        for (uint64_t e = g.off[u]; e < g.off[u + 1]; ++e) {
            const uint32_t v = g.to[e];
            if (v <= u) continue;
            const uint32_t cv = R.assign[v];
            if (cu == cv) {
                L.mat.push_back(cu);
                L.ii.push_back(static_cast<uint32_t>(u - R.comp_off[cu]));
                L.jj.push_back(v - R.comp_off[cv]);
                L.w.push_back(g.w[e]);
            } else {
                // endpoints of a cross edge are boundary vertices, whose
                // boundary id is base + local id (src/oracle.cpp:95-100)
                L.bi.push_back(static_cast<uint32_t>(R.bnd_off[cu] + (u - R.comp_off[cu])));
                L.bj.push_back(R.bnd_off[cv] + (v - R.comp_off[cv]));
                L.bw.push_back(g.w[e]);
            }
        }
    }
    return L;
}

template <class V>
std::vector<V> convert(const std::vector<double>& w, int shift) {
    std::vector<V> out(w.size());
    for (size_t i = 0; i < w.size(); ++i) out[i] = to_value<V>(w[i], shift);
    return out;
}

template <class V>
void scatter(MatArena& a, const std::vector<uint32_t>* mat, const std::vector<uint32_t>& ii,
             const std::vector<uint32_t>& jj, const std::vector<double>& w, int shift,
             cudaStream_t s) {
    if (ii.empty()) return;
    DBuf dm = mat ? upload(*mat, s) : DBuf();
    DBuf di = upload(ii, s), dj = upload(jj, s), dw = upload(convert<V>(w, shift), s);
    const uint64_t cnt = ii.size();
    scatter_pairs<V><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(
        a.view<V>(), mat ? dm.as<uint32_t>() : nullptr, di.as<uint32_t>(), dj.as<uint32_t>(),
        dw.as<V>(), cnt);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));  // keep staging buffers alive until consumed
}

struct EventTimer {
    cudaEvent_t a{}, b{};
    EventTimer() {
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
    }
    ~EventTimer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    void start(cudaStream_t s) { CK(cudaEventRecord(a, s)); }
    void stop(cudaStream_t s) { CK(cudaEventRecord(b, s)); }
    double ms() {
        CK(cudaEventSynchronize(b));
        float t = 0;
        CK(cudaEventElapsedTime(&t, a, b));
        return t;
    }
};

// Query-side tables and id maps on the device (shared by build and import).
// The id maps and the to-boundary arena, allocated and uploaded ahead of
// time: the build does it before K2, where device allocations are quick
// (right after K2 single small cudaMalloc calls have taken ~0.1 s each on
// these boxes, PSP_ALLOC_LOG), and finish_query_tables only fills them.
template <class V>
void alloc_query_tables(psp_gpu_oracle* o, cudaStream_t s) {
    const Reordered& R = o->R;
    const uint32_t k = R.k;
    if (o->d_cb.p && o->d_perm.p) return;
    std::vector<uint64_t> cb_off(k + 1, 0);
    for (uint32_t c = 0; c < k; ++c)
        cb_off[c + 1] = cb_off[c] + uint64_t(R.comp_off[c + 1] - R.comp_off[c]) *
                                        cb_stride(R.bnd_off[c + 1] - R.bnd_off[c]);
    o->d_cb.alloc(cb_off[k] * sizeof(V));
    o->d_cb_off = upload(cb_off, s);
    o->d_comp_off = upload(R.comp_off, s);
    o->d_perm = upload(R.perm, s);
    o->d_assign = upload(R.assign, s);
}

template <class V>
void finish_query_tables(psp_gpu_oracle* o, DBuf d_bnd, cudaStream_t s) {
    const uint32_t k = o->R.k;
    alloc_query_tables<V>(o, s);
    o->d_bnd_off = std::move(d_bnd);
    extract_to_boundary<V><<<std::max(k, 1u), 256, 0, s>>>(
        o->comps.view<V>(), o->d_comp_off.as<uint32_t>(), o->d_bnd_off.as<uint32_t>(),
        o->d_cb_off.as<uint64_t>(), o->d_cb.as<V>());
    CK_LAUNCH();
}

// Block query layout: every component pair block (c1 <= c2) of the
// boundary table stored contiguously as [column group][B1p rows][32
// columns], B1p = B1 rounded up to GK, INF in the padding. A 16-row chunk of
// one column group is then one 2 KB bulk copy for query_grouped instead of
// 144 address-computed 16-byte copies out of the tile arena. About 1.2x the
// symmetric arena; built only when it fits beside it with headroom.
template <class V>
__global__ void pack_query_blocks(const V* __restrict__ bg, uint32_t nb,
                                  const uint32_t* __restrict__ bnd_off, uint32_t k,
                                  const uint64_t* __restrict__ blk_off, V* __restrict__ bq) {
    const uint32_t c1 = blockIdx.x / k, c2 = blockIdx.x % k;
    if (c2 < c1) return;
    const uint32_t g1 = bnd_off[c1], B1 = bnd_off[c1 + 1] - g1;
    const uint32_t g2 = bnd_off[c2], B2 = bnd_off[c2 + 1] - g2;
    const uint64_t B1p = (B1 + GK - 1) / GK * GK, ncg = (B2 + 31) / 32;
    const uint64_t total = ncg * B1p * 32;
    V* out = bq + blk_off[blockIdx.x];
    for (uint64_t idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const uint64_t cg = idx / (B1p * 32), rem = idx - cg * B1p * 32;
        const uint32_t r = static_cast<uint32_t>(rem >> 5), col = static_cast<uint32_t>(cg * 32 + (rem & 31));
        out[idx] = (r < B1 && col < B2) ? bg[sym_off(g1 + r, g2 + col, nb)] : Ops<V>::inf();
    }
}

// Host half of build_query_blocks: the block offsets and the layout's
// allocation (no stream work, so the build runs it on a helper thread while
// K2 executes: the 48 GB cudaMalloc at cfg3 then costs no wall time).
// Returns the offsets, empty when the layout is not made.
// Block offsets of the layout (elements, per pair c1 <= c2); false when no
// layout is made (PSP_QUERY_LAYOUT=tiles, b == 0, k^2 past 31-bit keys).
bool query_block_offsets(const Reordered& R, std::vector<uint64_t>& off, uint64_t& elems) {
    const uint64_t k = R.k;
    off.clear();
    elems = 0;
    const char* lay = std::getenv("PSP_QUERY_LAYOUT");
    if (lay && std::strcmp(lay, "tiles") == 0) return false;
    if (R.b() == 0 || k * k >= (1ull << 31)) return false;
    off.assign(k * k, 0);
    for (uint64_t c1 = 0; c1 < k; ++c1) {
        const uint64_t B1 = R.bnd_off[c1 + 1] - R.bnd_off[c1], B1p = (B1 + GK - 1) / GK * GK;
        for (uint64_t c2 = c1; c2 < k; ++c2) {
            const uint64_t B2 = R.bnd_off[c2 + 1] - R.bnd_off[c2];
            off[c1 * k + c2] = elems;
            elems += (B2 + 31) / 32 * 32 * B1p;
        }
    }
    return true;
}

template <class V>
std::vector<uint64_t> plan_query_blocks(psp_gpu_oracle* o) {
    o->bq.reset();
    o->d_bq_off.reset();
    std::vector<uint64_t> off;
    uint64_t acc = 0;
    if (!query_block_offsets(o->R, off, acc)) return {};
    size_t free_b = 0, total_b = 0;
    mem_info(&free_b, &total_b);
    const uint64_t need = acc * sizeof(V) + off.size() * 8;
    if (need + (8ull << 30) > free_b) return {};  // keep 8 GB for query workspaces
    o->bq.alloc(acc * sizeof(V));
    return off;
}

// Device half: upload the offsets and pack the blocks from the finished
// reference-numbered boundary table.
template <class V>
void pack_query_layout(psp_gpu_oracle* o, const std::vector<uint64_t>& off, cudaStream_t s) {
    const uint64_t k = o->R.k;
    if (off.empty() || !o->bq.p || !o->bg.nmat) {
        o->bq.reset();
        return;
    }
    if (!o->d_bq_off.p || o->d_bq_off.bytes < off.size() * sizeof(uint64_t)) o->d_bq_off = upload(off, s);
    pack_query_blocks<V><<<unsigned(k * k), 256, 0, s>>>(o->bg.tiles.as<V>(), o->bg.nb[0],
                                                         o->d_bnd_off.as<uint32_t>(), uint32_t(k),
                                                         o->d_bq_off.as<uint64_t>(), o->bq.as<V>());
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
}

template <class V>
void build_query_blocks(psp_gpu_oracle* o, cudaStream_t s) {
    const std::vector<uint64_t> off = plan_query_blocks<V>(o);
    pack_query_layout<V>(o, off, s);
}

// The 16-bit residual layout of the boundary table for the u32 query
// product (query_kernels.cuh "16-bit residual product"): per pair block the
// saturated residuals (same [cg][B1p][32] geometry as the block layout, u16)
// and its potentials, per to-boundary row its 15-bit offsets and base. About
// half the block layout; built when it fits with 8 GB spare.
void build_query_blocks16(psp_gpu_oracle* o, cudaStream_t s) {
    const Reordered& R = o->R;
    const uint64_t k = R.k;
    o->bq16.reset();
    o->bqaux.reset();
    o->cb16.reset();
    o->d_rbase.reset();
    // opt-in (PSP_QUERY_U16=1): measured slower than the u32 product on cfg3
    // (31.3 vs 16.1 ms per 10M pairs, 0.7% of queries to the u32 fallback),
    // see DESIGN.md §3c
    const char* env = std::getenv("PSP_QUERY_U16");
    if (!(env && std::strcmp(env, "1") == 0)) return;
    if (o->kind.kind != PSP_VALUE_U32 || !o->bg.nmat || k * k >= (1ull << 31)) return;
    std::vector<uint64_t> off(k * k, 0), aoff(k * k, 0);
    uint64_t acc = 0, aacc = 0;
    uint32_t maxB = 1;
    for (uint64_t c1 = 0; c1 < k; ++c1) {
        const uint32_t B1 = R.bnd_off[c1 + 1] - R.bnd_off[c1];
        const uint64_t B1p = (B1 + GK - 1) / GK * GK;
        maxB = std::max(maxB, B1);
        for (uint64_t c2 = c1; c2 < k; ++c2) {
            const uint32_t B2 = R.bnd_off[c2 + 1] - R.bnd_off[c2];
            off[c1 * k + c2] = acc;
            acc += (B2 + 31) / 32 * 32 * B1p;
            aoff[c1 * k + c2] = aacc;
            aacc += (bqaux_words(B1, B2) + 3) / 4 * 4;  // 16-byte aligned
        }
    }
    size_t free_b = 0, total_b = 0;
    mem_info(&free_b, &total_b);
    const uint64_t need = acc * 2 + aacc * 4 + 2 * k * k * 8;
    if (need + (8ull << 30) > free_b) return;
    o->bq16.alloc(acc * 2);
    o->bqaux.alloc(aacc * 4);
    o->d_bq16_off = upload(off, s);
    o->d_aux_off = upload(aoff, s);
    // PSP_U16_SAT (tests only): a smaller saturation S sends most queries
    // through the lower-bound test and the u32 fallback
    const char* se = std::getenv("PSP_U16_SAT");
    o->u16_sat = se ? uint32_t(std::min<unsigned long>(std::strtoul(se, nullptr, 0), U16_SAT)) : U16_SAT;
    const size_t smem = size_t(2) * maxB * sizeof(uint32_t);
    if (smem > (48u << 10))
        CK(cudaFuncSetAttribute(pack_query_blocks16, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    pack_query_blocks16<<<unsigned(k * k), 256, smem, s>>>(
        o->bg.tiles.as<uint32_t>(), o->bg.nb[0], o->d_bnd_off.as<uint32_t>(), uint32_t(k),
        o->d_bq16_off.as<uint64_t>(), o->d_aux_off.as<uint64_t>(), o->bq16.as<uint16_t>(),
        o->bqaux.as<uint32_t>(), maxB, o->u16_sat);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
}

// K2 elimination order (bg_order.hpp) when the FW walks sparse tiles, the
// order beats the reference numbering, the unit count is small enough for
// the host simulation, and a second table fits for the permutation back
// (PSP_BG_ORDER=natural keeps the reference numbering, =component orders
// whole components). Fills posmap (boundary id -> K2 position).
// When the second table does not fit beside the component tables, those
// (idle during K2) are parked in host memory for the FW and the permutation
// (`spill`), if the host has room for them.
uint64_t host_mem_available() {
    std::ifstream f("/proc/meminfo");
    std::string key;
    uint64_t kb = 0;
    while (f >> key >> kb) {
        if (key == "MemAvailable:") return kb * 1024;
        f.ignore(256, '\n');
    }
    return 0;
}

// Memory-based layout choices (K1 grouping, the K2 order / packing / spill)
// select different NCCL call sequences, so with more than one rank every
// rank must take them from the same numbers: the minimum over ranks of each
// value (one small AllReduce on the build stream). A no-op on one GPU.
void agree_min(psp_gpu_ctx* ctx, uint64_t* vals, int count) {
    if (ctx->world <= 1) return;
    DBuf d(sizeof(uint64_t) * count);
    CK(cudaMemcpyAsync(d.p, vals, sizeof(uint64_t) * count, cudaMemcpyHostToDevice, ctx->stream));
    NCK(nccl().AllReduce(d.p, d.p, count, ncclUint64, ncclMin, ctx->comm, ctx->stream));
    CK(cudaMemcpyAsync(vals, d.p, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
}

// The host half of the K2 order (no device, no collective): units (pieces or
// components), the unit adjacency and the greedy elimination order. It only
// needs the reordered graph and its edge lists, so device_build runs it on a
// host thread while Phase 2 runs on the GPU.
struct BgPlan {
    bool use = false;          // an order that beats the reference numbering
    bool by_component = false;
    uint32_t nu = 0;
    std::vector<uint32_t> unit;
    std::vector<uint64_t> bsize;
    BgOrder ord;
};

BgPlan plan_bg_order(const Reordered& R, const EdgeLists& L) {
    BgPlan P;
    const uint32_t k = R.k;
    const uint64_t b = R.b();
    const char* env = std::getenv("PSP_BG_ORDER");
    const bool sparse = (b + T - 1) / T > 1 && std::getenv("PSP_FW_DENSE") == nullptr;
    if (!sparse || k < 2 || (env && std::strcmp(env, "natural") == 0)) return P;
    P.by_component = env && std::strcmp(env, "component") == 0;
    // unit of every boundary id: its component, or the connected part of
    // the component it lies in (union-find over the intra-component edges)
    std::vector<uint32_t>& unit = P.unit;
    unit.assign(b, 0);
    uint32_t nu = 0;
    if (P.by_component) {
        for (uint32_t c = 0; c < k; ++c)
            for (uint64_t i = R.bnd_off[c]; i < R.bnd_off[c + 1]; ++i) unit[i] = c;
        nu = k;
    } else {
        std::vector<uint32_t> up(R.n);
        for (uint64_t v = 0; v < R.n; ++v) up[v] = static_cast<uint32_t>(v);
        auto find = [&](uint32_t x) {
            while (up[x] != x) x = up[x] = up[up[x]];
            return x;
        };
        for (size_t e = 0; e < L.mat.size(); ++e) {
            const uint32_t base = static_cast<uint32_t>(R.comp_off[L.mat[e]]);
            const uint32_t x = find(base + L.ii[e]), y = find(base + L.jj[e]);
            if (x != y) up[std::max(x, y)] = std::min(x, y);
        }
        std::vector<uint32_t> id_of_root(R.n, UINT32_MAX);
        for (uint32_t c = 0; c < k; ++c)
            for (uint64_t i = R.bnd_off[c]; i < R.bnd_off[c + 1]; ++i) {
                // boundary vertices come first in their component (local id = i - bnd_off)
                const uint32_t r = find(static_cast<uint32_t>(R.comp_off[c] + (i - R.bnd_off[c])));
                if (id_of_root[r] == UINT32_MAX) id_of_root[r] = nu++;
                unit[i] = id_of_root[r];
            }
    }
    P.nu = nu;
    if (nu < 3 || nu > 16384) return P;
    P.bsize.assign(nu, 0);
    for (uint64_t i = 0; i < b; ++i) ++P.bsize[unit[i]];
    std::vector<std::pair<uint32_t, uint32_t>> adj;
    adj.reserve(L.bi.size());
    for (size_t e = 0; e < L.bi.size(); ++e) adj.emplace_back(unit[L.bi[e]], unit[L.bj[e]]);
    std::sort(adj.begin(), adj.end());
    adj.erase(std::unique(adj.begin(), adj.end()), adj.end());
    P.ord = bg_unit_order(nu, P.bsize, adj);
    bool ident = true;
    for (uint32_t i = 0; i < nu && ident; ++i) ident = P.ord.order[i] == i;
    if (std::getenv("PSP_FW_PROFILE"))
        std::fprintf(stderr, "[psp] K2 order over %u %s: simulated work %.3e (reference numbering %.3e)%s\n",
                     nu, P.by_component ? "components" : "pieces", P.ord.work, P.ord.natural,
                     ident ? ", kept" : "");
    P.use = !ident;
    return P;
}

// Chosen before the boundary-graph arena exists: `npos` is the working
// matrix size (positions incl. the tile-packing padding, >= b). Device
// memory must hold the working matrix with its panel plus the table in
// reference numbering (2 GB spare).
template <class V>
bool choose_bg_order(const psp_gpu_oracle* o, const BgPlan& plan, std::vector<uint32_t>& posmap,
                     uint64_t& npos, bool& spill) {
    const Reordered& R = o->R;
    const uint32_t k = R.k;
    const uint64_t b = R.b();
    spill = false;
    npos = b;
    const char* env = std::getenv("PSP_BG_ORDER");
    const bool sparse = (b + T - 1) / T > 1 && std::getenv("PSP_FW_DENSE") == nullptr;
    if (!sparse || k < 2 || (env && std::strcmp(env, "natural") == 0)) return false;
    size_t free_b = 0, total_b = 0;
    mem_info(&free_b, &total_b);
    // every rank decides from the smallest free device and host memory
    uint64_t agreed[2] = {free_b, host_mem_available()};
    agree_min(o->ctx, agreed, 2);
    free_b = agreed[0];
    const uint64_t host_avail = agreed[1];
    auto table_bytes = [](uint64_t n) {
        const uint64_t nb = (n + T - 1) / T;
        return ntiles_upper(uint32_t(nb)) * TT * sizeof(V);
    };
    // row-sharded storage: this rank's rows of the working matrix only, no
    // table in reference numbering (the shard gathers from the working one)
    const bool rows_only = o->row_storage;
    const uint64_t G = uint64_t(o->ctx->world);
    auto need = [&](uint64_t n) {
        if (rows_only)
            return table_bytes(n) / G + table_bytes(n) / (G * 8) + ((n + T - 1) / T + 1) * TT * sizeof(V) +
                   (2ull << 30);
        return table_bytes(n) + ((n + T - 1) / T + 1) * TT * sizeof(V) + table_bytes(b) + (2ull << 30);
    };
    if (!plan.use) return false;
    const std::vector<uint32_t>& unit = plan.unit;
    const std::vector<uint64_t>& bsize = plan.bsize;
    const BgOrder& ord = plan.ord;
    // positions: units in elimination order packed into tiles (bg_pack),
    // each unit's ids ascending; without room for the padding, contiguous
    std::vector<uint64_t> start;
    const char* pk = std::getenv("PSP_BG_PACK");
    // measured: cfg3 K2 8.29 -> 8.05 s, cfg2 unchanged; on small matrices
    // (a few tiles per side) the padding costs more than it saves
    // PSP_BG_PACK=0 turns packing off, PSP_BG_PACK=force turns it on at any
    // size (tests: small graphs exercise the padding positions bitwise)
    const bool force_pack = pk && std::strcmp(pk, "force") == 0;
    const bool pack = force_pack || (!(pk && std::strcmp(pk, "0") == 0) && b >= 128ull * T);
    npos = pack ? bg_pack(ord.order, bsize, T, 16, start) : bg_pack(ord.order, bsize, 1, 0, start);
    const uint64_t parked = o->comps.tiles.bytes;
    // room to park them: only PSP_K2_SPILL=host needs host memory (the
    // default drops the component tables and recomputes them after K2)
    const char* sp = std::getenv("PSP_K2_SPILL");
    const bool host_room = !(sp && std::strcmp(sp, "host") == 0) ||
                           host_avail >= parked + (8ull << 30);
    if (!force_pack && need(npos) > free_b && (need(npos) > free_b + parked || !host_room)) {
        npos = bg_pack(ord.order, bsize, 1, 0, start);  // contiguous
    }
    if (need(npos) > free_b) {
        if (rows_only || need(npos) > free_b + parked || !host_room) return false;
        spill = true;
    }
    // PSP_K2_FORCE_SPILL=1 (tests): take the spill path on any size
    if (std::getenv("PSP_K2_FORCE_SPILL") && !rows_only) spill = true;
    if (std::getenv("PSP_FW_PROFILE"))
        std::fprintf(stderr, "[psp] K2 layout: %llu positions for %llu boundary vertices%s\n",
                     (unsigned long long)npos, (unsigned long long)b, spill ? " (component tables off the device during K2)" : "");
    posmap.resize(b);
    for (uint64_t i = 0; i < b; ++i) posmap[i] = static_cast<uint32_t>(start[unit[i]]++);
    return true;
}

// ---- K1 with the nested-dissection elimination order (k1_order.hpp)
// Components [m0, m1) (this rank's range) are closed in groups sized to the
// free device memory: per group a working arena in FW positions, walked
// sparse, then permute_batch writes the tables in reference numbering into
// the final arena (which therefore needs no fill). Returns false (nothing
// done) when a single component's working arena does not fit.
struct K1Result {
    double init_ms = 0.0, k1_ms = 0.0, order_ms = 0.0;
    uint64_t walked_tiles = 0;
    std::string laps;  // host wall-clock laps (PSP_FW_PROFILE)
};

template <class V>
bool k1_ordered(psp_gpu_oracle* o, const EdgeLists& L, uint32_t m0, uint32_t m1, K1Result& res) {
    psp_gpu_ctx* ctx = o->ctx;
    cudaStream_t s = ctx->stream;
    const Reordered& R = o->R;
    const MatArena& F = o->comps;
    const int q = o->kind.shift;
    auto need = [&](uint32_t c) {  // working bytes of component c (tiles, panel, flags, lists)
        const uint64_t nb = F.nb[c];
        return (ntiles_upper(nb) * TT + nb * TT + nb) * sizeof(V) + 16 * nb + 64;
    };
    const auto tl = Clock::now();
    auto lap = [&](const char* what) {
        char buf[64];
        std::snprintf(buf, sizeof buf, " %s@%.1f", what, ms_since(tl));
        res.laps += buf;
    };
    size_t free_b = 0, total_b = 0;
    mem_info(&free_b, &total_b);
    lap("meminfo");
    // with several ranks the ordered path (and the AllReduce + range
    // broadcast behind it) is taken by all or none: agree on the smallest
    // free memory, then on every rank's range fitting the budget
    uint64_t fm = free_b;
    agree_min(ctx, &fm, 1);
    free_b = fm;
    const uint64_t margin = 1ull << 30;
    uint64_t fits = free_b >= margin;
    const uint64_t budget = fits ? free_b - margin : 0;
    for (uint32_t c = m0; c < m1 && fits; ++c)
        if (need(c) > budget) fits = 0;
    agree_min(ctx, &fits, 1);
    if (!fits) return false;
    const auto t0 = Clock::now();
    // intra-component edges bucketed by component
    std::vector<uint64_t> eoff(R.k + 1, 0);
    for (uint32_t c : L.mat) ++eoff[c + 1];
    for (uint32_t c = 0; c < R.k; ++c) eoff[c + 1] += eoff[c];
    std::vector<uint64_t> eidx(L.mat.size());
    {
        std::vector<uint64_t> fill(eoff.begin(), eoff.end() - 1);
        for (uint64_t e = 0; e < L.mat.size(); ++e) eidx[fill[L.mat[e]]++] = e;
    }
    // positions per component, on all host threads
    std::vector<uint64_t> pos_off(m1 - m0 + 1, 0);
    for (uint32_t c = m0; c < m1; ++c)
        pos_off[c - m0 + 1] = pos_off[c - m0] + (R.comp_off[c + 1] - R.comp_off[c]);
    std::vector<uint32_t> pos(pos_off.back());
    {
        std::atomic<uint32_t> next{m0};
        const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t)
            pool.emplace_back([&] {
                NdOrder nd;
                std::vector<std::pair<uint32_t, uint32_t>> edges;
                for (uint32_t c; (c = next.fetch_add(1)) < m1;) {
                    const uint32_t n = R.comp_off[c + 1] - R.comp_off[c];
                    edges.clear();
                    for (uint64_t x = eoff[c]; x < eoff[c + 1]; ++x)
                        edges.emplace_back(L.ii[eidx[x]], L.jj[eidx[x]]);
                    const std::vector<uint32_t> p = nd.positions(n, edges);
                    std::copy(p.begin(), p.end(), pos.begin() + pos_off[c - m0]);
                }
            });
        for (auto& th : pool) th.join();
    }
    res.order_ms += ms_since(t0);
    lap("ordered");
    EventTimer t_init, t_fw;
    for (uint32_t g0 = m0; g0 < m1;) {
        uint32_t g1 = g0;
        uint64_t bytes = 0;
        while (g1 < m1 && bytes + need(g1) <= budget) bytes += need(g1++);
        std::vector<uint64_t> gsizes(g1 - g0);
        for (uint32_t c = g0; c < g1; ++c) gsizes[c - g0] = R.comp_off[c + 1] - R.comp_off[c];
        std::vector<uint32_t> gm, gi, gj;
        std::vector<double> gw;
        for (uint32_t c = g0; c < g1; ++c) {
            const uint32_t* pc = pos.data() + pos_off[c - m0];
            for (uint64_t x = eoff[c]; x < eoff[c + 1]; ++x) {
                const uint64_t e = eidx[x];
                gm.push_back(c - g0);
                gi.push_back(pc[L.ii[e]]);
                gj.push_back(pc[L.jj[e]]);
                gw.push_back(L.w[e]);
            }
        }
        std::vector<uint64_t> goff(g1 - g0 + 1);
        for (uint32_t c = g0; c <= g1; ++c) goff[c - g0] = pos_off[c - m0] - pos_off[g0 - m0];
        std::vector<uint32_t> gpos(pos.begin() + pos_off[g0 - m0], pos.begin() + pos_off[g1 - m0]);
        lap("host-lists");
        MatArena W;
        W.create(gsizes, sizeof(V), true, s, 1);
        lap("W-alloc");
        t_init.start(s);
        fill_arena<V>(W, s, ctx->sms);
        scatter<V>(W, &gm, gi, gj, gw, q, s);
        t_init.stop(s);
        res.init_ms += t_init.ms();
        lap("init");
        DBuf d_pos = upload(gpos, s), d_off = upload(goff, s);
        t_fw.start(s);
        run_fw<V>(W, s, ctx->sms);
        if (W.nb_max > 0) {
            permute_batch<V><<<dim3(W.nb_max, W.nb_max, g1 - g0), 256, 0, s>>>(
                W.view<V>(), F.view<V>(), g0, d_pos.as<uint32_t>(), d_off.as<uint64_t>());
            CK_LAUNCH();
        }
        t_fw.stop(s);
        res.k1_ms += t_fw.ms();
        lap("fw");
        res.walked_tiles += W.sparse ? W.walked_tiles : W.relaxations() / (uint64_t(T) * T * T);
        g0 = g1;
    }
    lap("W-freed");
    return true;
}

template <class V>
void device_build(psp_gpu_oracle* o, psp_build_stats* st) {
    psp_gpu_ctx* ctx = o->ctx;
    cudaStream_t s = ctx->stream;
    const Reordered& R = o->R;
    const uint32_t k = R.k;
    const int q = o->kind.shift;
    EventTimer t_k2, t_post;

    // ---- Phase 2: K0 + K1
    auto t0 = Clock::now();
    std::vector<uint64_t> sizes(k);
    for (uint32_t c = 0; c < k; ++c) sizes[c] = R.comp_off[c + 1] - R.comp_off[c];
    EdgeLists L = split_edges(R);
    const double split_ms = ms_since(t0);
    double init_ms = 0.0, k1_ms = 0.0, order_ms = 0.0;
    uint64_t k1_relax = 0;
    double create_ms = 0.0;
    std::string k1_laps;
    const char* k1env = std::getenv("PSP_K1_ORDER");
    const bool want_order = !(k1env && std::strcmp(k1env, "natural") == 0);
    bool ordered = false;
    // Phase 2 as a unit: also re-run after K2 when the component tables had
    // to leave the device for the boundary-graph FW (`spill`, see below)
    // force: -1 free choice, 0 dense walk, 1 ordered (the spill recompute
    // must take the path that produced the tables K2 was seeded from, or
    // f32 tables could round differently)
    auto phase2 = [&](int force) {
        ordered = false;
        // this rank's components (all of them on one GPU)
        std::vector<uint32_t> cut{0, k};
        if (want_order && force != 0) {
            const auto tc = Clock::now();
            o->comps.create(sizes, sizeof(V), false, s);
            create_ms = ms_since(tc);
            if (ctx->world > 1) cut = k1_ranges(o->comps, ctx->world);
            if (o->comps.nb_max > 2) {
                K1Result res;
                ordered = k1_ordered<V>(o, L, cut[ctx->rank], cut[ctx->rank + 1], res);
                init_ms = res.init_ms;
                k1_ms = res.k1_ms;
                order_ms = res.order_ms;
                k1_relax = res.walked_tiles;
                k1_laps = res.laps;
            }
            if (ordered) {
                if (ctx->world > 1) {
                    // k1_relax: this rank's share; total over ranks
                    DBuf d_w(sizeof(unsigned long long));
                    CK(cudaMemcpyAsync(d_w.p, &k1_relax, 8, cudaMemcpyHostToDevice, s));
                    NCK(nccl().AllReduce(d_w.p, d_w.p, 1, ncclUint64, ncclSum, ctx->comm, s));
                    EventTimer t_bc;
                    t_bc.start(s);
                    broadcast_component_ranges<V>(o->comps, cut, ctx);
                    t_bc.stop(s);
                    k1_ms += t_bc.ms();
                    CK(cudaMemcpyAsync(&k1_relax, d_w.p, 8, cudaMemcpyDeviceToHost, s));
                    CK(cudaStreamSynchronize(s));
                }
                k1_relax *= uint64_t(T) * T * T;
            }
        }
        if (force == 1 && !ordered)
            throw Fail{PSP_ENOMEM, "component tables recomputed after K2: the nested-dissection "
                                   "path that built them no longer fits beside the boundary-graph "
                                   "table (set PSP_K2_SPILL=host)"};
        if (!ordered) {  // reference numbering, dense walk, in place
            EventTimer t_init, t_k1;
            o->comps.create(sizes, sizeof(V), true, s);
            t_init.start(s);
            fill_arena<V>(o->comps, s, ctx->sms);
            scatter<V>(o->comps, &L.mat, L.ii, L.jj, L.w, q, s);
            t_init.stop(s);
            t_k1.start(s);
            if (ctx->world > 1) run_fw_components_sharded<V>(o->comps, ctx);
            else run_fw<V>(o->comps, s, ctx->sms);
            t_k1.stop(s);
            CK(cudaStreamSynchronize(s));
            o->comps.panel.reset();  // K1 scratch
            k1_ms = t_k1.ms();
            init_ms = t_init.ms();
            k1_relax = o->comps.relaxations();
        }
    };
    // the K2 elimination order needs only host data: plan it on a host
    // thread while Phase 2 runs on the device
    BgPlan plan;
    std::exception_ptr plan_err;
    double plan_ms = 0.0;
    std::thread planner([&] {
        try {
            const auto tp = Clock::now();
            plan = plan_bg_order(R, L);
            plan_ms = ms_since(tp);
        } catch (...) {
            plan_err = std::current_exception();
        }
    });
    struct PlanJoin {
        std::thread& t;
        ~PlanJoin() {
            if (t.joinable()) t.join();
        }
    } plan_join{planner};
    phase2(-1);
    const bool first_ordered = ordered;
    const double component_ms = ms_since(t0);
    if (std::getenv("PSP_FW_PROFILE"))
        std::fprintf(stderr,
                     "[psp] component phase %.1f ms (%s): split %.1f, order %.1f, device init "
                     "%.2f + K1 %.2f ms, %.3e relaxations; table alloc %.1f ms, laps:%s\n",
                     component_ms, ordered ? "nested-dissection order, sparse walk" : "dense walk",
                     split_ms, order_ms, init_ms, k1_ms, double(k1_relax), create_ms,
                     k1_laps.c_str());

    // ---- Phase 3: BG init + K2 + query tables
    std::vector<uint64_t> bq_off;
    uint64_t bq_elems = 0;
    DBuf bq_reused;
    std::exception_ptr bq_err;
    std::thread bq_planner;
    struct BqJoin {
        std::thread& t;
        ~BqJoin() {
            if (t.joinable()) t.join();
        }
    } bq_join{bq_planner};
    bool bq_planned = false;
    t0 = Clock::now();
    const bool prof = std::getenv("PSP_FW_PROFILE") != nullptr;
    auto lap = [&](const char* what) {  // PSP_FW_PROFILE: synchronised wall-clock laps
        if (!prof) return;
        CK(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[psp] boundary lap: %s at %.1f ms\n", what, ms_since(t0));
    };
    const uint64_t b = R.b();
    DBuf d_bnd = upload(R.bnd_off, s);
    unsigned long long clique = 0;
    double k2_ms = 0.0, bg_order_ms = 0.0;
    uint64_t k2_relax = 0, k2_npos = b;
    bool k2_permuted = false, k2_spill = false;
    if (b > 0) {
        t_post.start(s);
        // K2 elimination order (bg_order.hpp): boundary id i sits at
        // posmap[i] of the npos-vertex working matrix during the FW; P ->
        // reference ids afterwards
        std::vector<uint32_t> posmap;
        bool spill = false;
        uint64_t npos = b;
        const auto tord = Clock::now();
        planner.join();
        if (plan_err) std::rethrow_exception(plan_err);
        const bool permuted = choose_bg_order<V>(o, plan, posmap, npos, spill);
        bg_order_ms = ms_since(tord);  // on the critical path (the plan overlapped Phase 2)
        (void)plan_ms;
        k2_npos = permuted ? npos : b;
        k2_permuted = permuted;
        k2_spill = spill;
        const int row_shard[3] = {ctx->device, ctx->rank, ctx->world};
        // ordered K2: its working matrix dies right after the permutation, when
        // the block layout is packed -- one allocation serves both (no 40 GB
        // cudaFree + 48 GB cudaMalloc between K2 and the layout; such calls
        // have stalled for up to 0.18 s on these boxes)
        bool reuse_bq = false;
        if (permuted && !spill && !o->row_storage && query_block_offsets(R, bq_off, bq_elems)) {
            const uint64_t work = ntiles_upper(uint32_t((npos + T - 1) / T)) * TT * sizeof(V);
            const uint64_t lay = bq_elems * sizeof(V);
            size_t free_b = 0, total_b = 0;
            mem_info(&free_b, &total_b);
            const uint64_t table = ntiles_upper(uint32_t((b + T - 1) / T)) * TT * sizeof(V);
            const uint64_t panel = ((npos + T - 1) / T + 1) * TT * sizeof(V);
            reuse_bq = std::max(work, lay) + table + panel + (10ull << 30) <= free_b;
            o->bg.min_tile_bytes = reuse_bq ? lay : 0;
        }
        if (!reuse_bq) bq_off.clear();
        o->bg.create({permuted ? npos : b}, sizeof(V), true, s, -1, o->row_storage ? row_shard : nullptr);
        o->bg.min_tile_bytes = 0;
        if (std::getenv("PSP_FW_PROFILE"))
            std::fprintf(stderr, "[psp] boundary phase: order chosen at %.1f ms\n", ms_since(t0));
        if (!permuted) {
            posmap.resize(b);
            for (uint64_t i = 0; i < b; ++i) posmap[i] = static_cast<uint32_t>(i);
        }
        lap("table allocated");
        fill_arena<V>(o->bg, s, ctx->sms);
        lap("table filled");
        DBuf d_pos = upload(posmap, s);
        DBuf d_clique(sizeof(unsigned long long));
        CK(cudaMemsetAsync(d_clique.p, 0, sizeof(unsigned long long), s));
        copy_boundary_blocks<V><<<k, 256, 0, s>>>(o->comps.view<V>(), d_bnd.as<uint32_t>(),
                                                  d_pos.as<uint32_t>(), o->bg.view<V>(),
                                                  d_clique.as<unsigned long long>());
        CK_LAUNCH();
        if (permuted) {
            std::vector<uint32_t> pi(L.bi.size()), pj(L.bj.size());
            for (size_t e = 0; e < pi.size(); ++e) {
                pi[e] = posmap[L.bi[e]];
                pj[e] = posmap[L.bj[e]];
            }
            scatter<V>(o->bg, nullptr, pi, pj, L.bw, q, s);
        } else {
            scatter<V>(o->bg, nullptr, L.bi, L.bj, L.bw, q, s);
        }
        CK(cudaMemcpyAsync(&clique, d_clique.p, sizeof(clique), cudaMemcpyDeviceToHost, s));
        t_post.stop(s);
        lap("edges scattered");
        CK(cudaStreamSynchronize(s));
        init_ms += t_post.ms();
        // `spill`: the component tables leave the device for K2. Default:
        // dropped and recomputed afterwards (Phase 2 again: host order +
        // init + K1, ~1 s on cfg4, NVLink broadcast of the ranges when
        // sharded). PSP_K2_SPILL=host parks them in host memory instead
        // (copied on side streams from a helper thread, overlapping the FW),
        // which costs a PCIe round trip of the whole arena, shared by all
        // ranks of a node.
        const char* spill_env = std::getenv("PSP_K2_SPILL");
        const bool park_host = spill && spill_env && std::strcmp(spill_env, "host") == 0;
        const bool recompute = spill && !park_host;
        if (recompute) o->comps = MatArena();
        std::unique_ptr<unsigned char[]> parked;  // default-initialised: no 70 GB memset
        size_t parked_bytes = 0;
        std::thread parker;
        struct Joiner {
            std::thread& t;
            ~Joiner() {
                if (t.joinable()) t.join();
            }
        } join_on_unwind{parker};
        Fail park_fail{PSP_OK, ""};
        if (park_host) {
            parked_bytes = o->comps.tiles.bytes;
            parked.reset(new unsigned char[parked_bytes]);
            parker = std::thread([&] {
                try {
                    staged_copy(parked.get(), o->comps.tiles.p, parked_bytes, true, ctx->device);
                } catch (const Fail& f) {
                    park_fail = f;
                }
            });
        }
        // the table in reference numbering: allocated up front (no host
        // allocation stalls inside the K2 window) unless the component
        // tables must leave the device first
        MatArena ref;
        if (permuted && !spill && !o->row_storage) ref.create({b}, sizeof(V), false, s);
        // query-side buffers now, while allocations are quick (see
        // alloc_query_tables); the spill path frees the component tables
        // first and allocates after K2 as before
        if (!spill) {
            uint64_t cb_elems = 0;
            for (uint32_t c = 0; c < k; ++c)
                cb_elems += uint64_t(R.comp_off[c + 1] - R.comp_off[c]) *
                            cb_stride(R.bnd_off[c + 1] - R.bnd_off[c]);
            size_t free_b = 0, total_b = 0;
            mem_info(&free_b, &total_b);
            if (cb_elems * sizeof(V) + (4ull << 30) < free_b) {  // else after K2, as before
                alloc_query_tables<V>(o, s);
                if (reuse_bq) o->d_bq_off = upload(bq_off, s);
            }
        }
        // the block query layout's offsets and allocation on a helper thread
        // while K2 runs (not beside spilled component tables: the memory is
        // K2's then)
        if (!o->row_storage && !spill && !reuse_bq) {
            bq_planner = std::thread([&, dev = ctx->device] {
                try {
                    CK(cudaSetDevice(dev));
                    bq_off = plan_query_blocks<V>(o);
                } catch (...) {
                    bq_err = std::current_exception();
                }
            });
        }
        t_k2.start(s);
        if (ctx->world > 1) run_fw_sharded<V>(o->bg, ctx);
        else run_fw<V>(o->bg, s, ctx->sms);
        k2_relax = o->bg.relaxations();  // (reads the walked-tile count: syncs)
        const double fw_done_ms = ms_since(t0);
        if (park_host) {
            parker.join();
            if (park_fail.st != PSP_OK) throw park_fail;
            o->comps.tiles.reset();
        }
        if (o->row_storage) {
            // the working matrix stays distributed (rows of this rank), with
            // its position map, for psp_gpu_shard_create to gather from
            t_k2.stop(s);
            o->bg.panel.reset();
            o->d_bg_pos = std::move(d_pos);
        } else if (permuted) {
            const double p0 = ms_since(t0);
            if (spill) {
                o->bg.panel.reset();
                ref.create({b}, sizeof(V), false, s);
            }
            const double p1 = ms_since(t0);
            const uint32_t nb = ref.nb[0];
            permute_sym<V><<<dim3(nb, nb), 256, 0, s>>>(o->bg.tiles.as<V>(), o->bg.nb[0],
                                                        ref.tiles.as<V>(), nb, uint32_t(b),
                                                        d_pos.as<uint32_t>());
            CK_LAUNCH();
            if (!spill) t_k2.stop(s);
            CK(cudaStreamSynchronize(s));
            const double p2 = ms_since(t0);
            o->bg.panel.reset();
            if (reuse_bq) bq_reused = std::move(o->bg.tiles);  // becomes the block layout
            o->bg = std::move(ref);
            if (std::getenv("PSP_FW_PROFILE"))
                std::fprintf(stderr,
                             "[psp] K2 permutation: alloc %.1f ms, permute_sym %.1f ms, frees %.1f ms\n",
                             p1 - p0, p2 - p1, ms_since(t0) - p2);
        }
        if (recompute) {  // the component tables come back: Phase 2 again
            const double back0 = ms_since(t0);
            const double si = init_ms, sk = k1_ms, so = order_ms;
            const uint64_t sr = k1_relax;
            const double sc = create_ms;
            const std::string sl = k1_laps;
            phase2(first_ordered ? 1 : 0);
            init_ms = si, k1_ms = sk, order_ms = so, k1_relax = sr, create_ms = sc;
            k1_laps = sl;
            if (std::getenv("PSP_FW_PROFILE"))
                std::fprintf(stderr,
                             "[psp] component tables dropped during K2: FW done at %.0f ms, "
                             "recomputed in %.0f ms (boundary phase so far %.0f ms)\n",
                             fw_done_ms, ms_since(t0) - back0, ms_since(t0));
        }
        if (park_host) {  // the component tables come back
            const double back0 = ms_since(t0);
            o->comps.tiles.alloc(parked_bytes);
            CK(cudaStreamSynchronize(s));
            staged_copy(o->comps.tiles.p, parked.get(), parked_bytes, false, ctx->device);
            if (std::getenv("PSP_FW_PROFILE"))
                std::fprintf(stderr,
                             "[psp] component tables parked on the host during K2 (%.1f GB): FW done "
                             "at %.0f ms, copy back %.0f ms (boundary phase so far %.0f ms)\n",
                             parked_bytes / 1e9, fw_done_ms, ms_since(t0) - back0, ms_since(t0));
        }
        if (!o->row_storage && (!permuted || spill)) t_k2.stop(s);
        CK(cudaStreamSynchronize(s));
        k2_ms = t_k2.ms();
        if (std::getenv("PSP_FW_PROFILE"))
            std::fprintf(stderr,
                         "[psp] boundary phase: FW issued+done at %.1f ms, K2 (FW + permute) %.1f "
                         "ms device, phase so far %.1f ms\n",
                         fw_done_ms, k2_ms, ms_since(t0));
    }
    // query-side tables
    lap("K2 done");
    t_post.start(s);
    finish_query_tables<V>(o, std::move(d_bnd), s);
    t_post.stop(s);
    CK(cudaStreamSynchronize(s));
    init_ms += t_post.ms();
    lap("to-boundary tables");
    // panels are build-time scratch
    o->comps.panel.reset();
    o->bg.panel.reset();
    lap("panels freed");
    if (!o->row_storage) {  // replicated queries only
        if (bq_planner.joinable()) {
            bq_planner.join();
            if (bq_err) std::rethrow_exception(bq_err);
            bq_planned = !bq_off.empty();  // else retried below, with K2's scratch freed
        }
        if (bq_reused.p) {
            o->bq = std::move(bq_reused);
            bq_planned = true;
        }
        if (!bq_planned) bq_off = plan_query_blocks<V>(o);
        pack_query_layout<V>(o, bq_off, s);
        lap("block layout");
        build_query_blocks16(o, s);
    }
    const double boundary_ms = ms_since(t0);

    o->device_bytes = o->comps.bytes() + o->bg.bytes() + o->d_cb.bytes + o->d_cb_off.bytes +
                      o->d_comp_off.bytes + o->d_bnd_off.bytes + o->d_perm.bytes +
                      o->d_assign.bytes + o->bq.bytes + o->d_bq_off.bytes + o->bq16.bytes +
                      o->bqaux.bytes + o->cb16.bytes + o->d_rbase.bytes;
    if (st) {
        st->component_apsp_ms = component_ms;
        st->boundary_ms = boundary_ms;
        st->k1_device_ms = k1_ms;
        st->k2_device_ms = k2_ms;
        st->init_device_ms = init_ms;
        st->k1_relaxations = k1_relax;
        st->k2_relaxations = k2_relax;
        st->boundary_total = b;
        st->bg_edges = L.bi.size() + clique;
        uint64_t stored = 0;
        for (uint32_t c = 0; c < k; ++c)
            stored += sizes[c] * sizes[c] + (R.bnd_off[c + 1] - R.bnd_off[c]) * b;
        st->stored_entries = stored;
        st->value_kind = o->kind.kind;
        st->fixed_point_shift = o->kind.shift;
        st->device_bytes = o->device_bytes;
        st->k2_positions = k2_npos;
        st->k2_order = k2_permuted ? 1 : 0;
        st->k2_spilled = k2_spill ? 1 : 0;
        st->split_ms = split_ms;
        st->k1_order_ms = order_ms;
        st->bg_order_ms = bg_order_ms;
    }
}

// The id maps of an imported / loaded oracle (validated as
// psp_gpu_oracle_import documents).
void reordered_from_ids(Reordered& R, uint64_t n, uint32_t k, const uint32_t* permutation,
                        const uint32_t* assignment, const uint64_t* component_offset,
                        const uint64_t* boundary_offset) {
    R.n = n;
    R.k = k;
    R.perm.assign(permutation, permutation + n);
    R.inv.assign(n, 0);
    std::vector<uint8_t> seen(n, 0);
    for (uint64_t v = 0; v < n; ++v) {
        if (R.perm[v] >= n || seen[R.perm[v]]++) throw ArgError("oracle_import: bad permutation");
        R.inv[R.perm[v]] = static_cast<uint32_t>(v);
    }
    R.assign.assign(assignment, assignment + n);
    R.comp_off.resize(k + 1);
    R.bnd_off.resize(k + 1);
    for (uint32_t c = 0; c <= k; ++c) {
        R.comp_off[c] = static_cast<uint32_t>(component_offset[c]);
        R.bnd_off[c] = static_cast<uint32_t>(boundary_offset[c]);
    }
    if (R.comp_off[0] != 0 || R.comp_off[k] != n || R.bnd_off[0] != 0)
        throw ArgError("oracle_import: offsets do not cover the graph");
    R.flags.assign(n, 0);
    for (uint32_t c = 0; c < k; ++c) {
        const uint32_t s = R.comp_off[c + 1] - R.comp_off[c];
        const uint32_t bc = R.bnd_off[c + 1] - R.bnd_off[c];
        if (R.comp_off[c + 1] < R.comp_off[c] || R.bnd_off[c + 1] < R.bnd_off[c] || bc > s)
            throw ArgError("oracle_import: inconsistent offsets");
        for (uint32_t i = 0; i < s; ++i) {
            if (R.assign[R.comp_off[c] + i] != c) throw ArgError("oracle_import: assignment/offset mismatch");
            R.flags[R.comp_off[c] + i] = i < bc;  // boundary-first local ids
        }
    }
}

// Kind for imported tables: u32 when every finite entry is exact in fixed
// point 2^q (q <= 24) below INF, else f32.
Kind choose_kind_tables(int requested, const std::vector<const double*>& ptr,
                        const std::vector<uint64_t>& len) {
    if (requested == PSP_VALUE_F32) return {PSP_VALUE_F32, 0};
    double maxv = 0.0;
    for (size_t t = 0; t < ptr.size(); ++t)
        for (uint64_t i = 0; i < len[t]; ++i)
            if (std::isfinite(ptr[t][i])) maxv = std::max(maxv, ptr[t][i]);
    for (int q = 0; q <= 24; ++q) {
        const double scale = std::ldexp(1.0, q);
        if (2.0 * maxv * scale >= double(U32_INF)) break;
        bool ok = true;
        for (size_t t = 0; t < ptr.size() && ok; ++t)
            for (uint64_t i = 0; i < len[t] && ok; ++i) {
                const double x = ptr[t][i];
                if (std::isinf(x)) continue;
                if (!(x >= 0) || std::floor(x * scale) != x * scale) ok = false;
            }
        if (ok) return {PSP_VALUE_U32, q};
    }
    if (requested == PSP_VALUE_U32)
        throw Fail{PSP_EOVERFLOW, "import: tables are not exact in u32 fixed point"};
    return {PSP_VALUE_F32, 0};
}

// Query-side tables of an imported or loaded oracle.
template <class V>
void finish_import(psp_gpu_oracle* o) {
    cudaStream_t s = o->ctx->stream;
    finish_query_tables<V>(o, upload(o->R.bnd_off, s), s);
    CK(cudaStreamSynchronize(s));
    build_query_blocks<V>(o, s);
    build_query_blocks16(o, s);
    o->device_bytes = o->comps.bytes() + o->bg.bytes() + o->d_cb.bytes + o->bq.bytes + o->bq16.bytes +
                      o->bqaux.bytes + o->cb16.bytes;
}

template <class V>
void import_tables(psp_gpu_oracle* o, const double* const* ct, const double* const* bt) {
    cudaStream_t s = o->ctx->stream;
    const Reordered& R = o->R;
    const uint32_t k = R.k;
    const uint64_t b = R.b();
    std::vector<uint64_t> sizes(k);
    for (uint32_t c = 0; c < k; ++c) sizes[c] = R.comp_off[c + 1] - R.comp_off[c];
    o->comps.create(sizes, sizeof(V), false, s);
    fill_arena<V>(o->comps, s, o->ctx->sms);
    auto to_v = [&](const double* src, uint64_t cnt) {
        std::vector<V> h(cnt);
        for (uint64_t i = 0; i < cnt; ++i)
            h[i] = std::isinf(src[i]) ? Ops<V>::inf() : to_value<V>(src[i], o->kind.shift);
        return h;
    };
    for (uint32_t c = 0; c < k; ++c) {
        const uint64_t cnt = sizes[c] * sizes[c];
        if (!cnt) continue;
        DBuf d = upload(to_v(ct[c], cnt), s);
        pack_window<V><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(o->comps.view<V>(), c, 0,
                                                                   uint32_t(sizes[c]),
                                                                   uint32_t(sizes[c]), d.as<V>());
        CK_LAUNCH();
        CK(cudaStreamSynchronize(s));
    }
    if (b > 0) {
        o->bg.create({b}, sizeof(V), false, s);
        fill_arena<V>(o->bg, s, o->ctx->sms);
        for (uint32_t c = 0; c < k; ++c) {
            const uint64_t rows = R.bnd_off[c + 1] - R.bnd_off[c], cnt = rows * b;
            if (!cnt) continue;
            DBuf d = upload(to_v(bt[c], cnt), s);
            pack_window<V><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(
                o->bg.view<V>(), 0, R.bnd_off[c], uint32_t(rows), uint32_t(b), d.as<V>());
            CK_LAUNCH();
            CK(cudaStreamSynchronize(s));
        }
    }
    finish_import<V>(o);
}

void set_peak_entries(const Reordered& R, unsigned workers, psp_build_stats* st) {
    if (!st) return;
    // RoundRobin placement over min(workers, k) (src/oracle.cpp:181-191)
    const uint32_t p = std::max<uint32_t>(1, std::min<uint32_t>(workers, R.k));
    std::vector<uint64_t> per(p, 0);
    for (uint32_t c = 0; c < R.k; ++c) {
        const uint64_t s = R.comp_off[c + 1] - R.comp_off[c];
        per[c % p] += s * s + (R.bnd_off[c + 1] - R.bnd_off[c]) * R.b();
    }
    st->peak_table_entries_per_worker = *std::max_element(per.begin(), per.end());
}

psp_gpu_oracle* build_from_csr(psp_gpu_ctx* ctx, const Csr& g, uint32_t k,
                               const std::vector<uint32_t>& assignment, const double* ew,
                               uint64_t m, int value_kind, double partition_ms,
                               psp_build_stats* st) {
    auto o = std::make_unique<psp_gpu_oracle>();
    o->ctx = ctx;
    o->kind = choose_kind(value_kind, ew, m, g.n);
    o->scale = std::ldexp(1.0, -o->kind.shift);
    auto t0 = Clock::now();
    o->R = reorder(g, k, assignment);
    if (st) {
        std::memset(st, 0, sizeof(*st));
        st->partition_ms = partition_ms + ms_since(t0);
    }
    CK(cudaSetDevice(ctx->device));
    o->row_storage = ctx->storage == PSP_STORAGE_ROW_SHARDED && ctx->world > 1;
    if (o->kind.kind == PSP_VALUE_U32) device_build<uint32_t>(o.get(), st);
    else device_build<float>(o.get(), st);
    return o.release();
}

template <class V>
void dense_apsp(psp_gpu_ctx* ctx, const Csr& g, const double* ew, uint64_t m, Kind kind,
                double* out) {
    cudaStream_t s = ctx->stream;
    const uint64_t n = g.n;
    if (n == 0) return;
    if (n > 0xffffffffull / 2) throw ArgError("apsp: vertex count too large");
    MatArena a;
    a.create({n}, sizeof(V), true, s);
    fill_arena<V>(a, s, ctx->sms);
    std::vector<uint32_t> ii, jj;
    std::vector<double> w;
    for (uint64_t u = 0; u < n; ++u)
        for (uint64_t e = g.off[u]; e < g.off[u + 1]; ++e)
            if (g.to[e] > u) {
                ii.push_back(static_cast<uint32_t>(u));
                jj.push_back(g.to[e]);
                w.push_back(g.w[e]);
            }
    (void)ew;
    (void)m;
    scatter<V>(a, nullptr, ii, jj, w, kind.shift, s);
    run_fw<V>(a, s, ctx->sms);
    DBuf d(n * n * sizeof(V));
    const uint64_t cnt = n * n;
    unpack_window<V><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(a.view<V>(), 0, 0, uint32_t(n), 0,
                                                                 uint32_t(n), d.as<V>());
    CK_LAUNCH();
    std::vector<V> h(cnt);
    CK(cudaMemcpyAsync(h.data(), d.p, cnt * sizeof(V), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    to_f64(h, out, std::ldexp(1.0, -kind.shift));
}

template <class V>
void export_window(const psp_gpu_oracle* o, const MatArena& a, uint32_t m, uint32_t row0,
                   uint32_t nrows, uint32_t ncols, double* dst) {
    const uint64_t cnt = uint64_t(nrows) * ncols;
    if (cnt == 0) return;
    cudaStream_t s = o->ctx->stream;
    CK(cudaSetDevice(o->ctx->device));
    DBuf d(cnt * sizeof(V));
    unpack_window<V><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(a.view<V>(), m, row0, nrows, 0,
                                                                 ncols, d.as<V>());
    CK_LAUNCH();
    std::vector<V> h(cnt);
    CK(cudaMemcpyAsync(h.data(), d.p, cnt * sizeof(V), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    to_f64(h, dst, o->scale);
}

// Sparse grouping when count * SPARSE_GROUPING_RATIO < k^2 and k^2 is large.
// Measured on cfg3 (k^2 = 1,048,576 bins, profiles/r2/query_kernel_sweep_cfg3.jsonl):
// 1K pairs 12.9 (sparse) vs 12.7 (dense) M queries/s, 10K 38.7 vs 46.7, 100K
// 70.9 vs 71.3: the k^2 passes are not what small batches wait on there (their
// blocks are read with no reuse, and the per-task chunk pipeline is latency
// bound), so the dense path stays up to 2^24 bins (k = 4096, 268 MB of bins).
constexpr uint64_t SPARSE_GROUPING_RATIO = 4;
constexpr uint64_t SPARSE_GROUPING_MIN_BINS = uint64_t(1) << 24;

// Counting sort by component pair, task records, query_grouped, finish.
// `bnd_off` is the host copy of the boundary offsets (task-count bound).
template <class V, int MODE>
void launch_grouped(GroupWorkspace& gw, const std::vector<uint32_t>& bnd_off, int sms,
                    const QueryView<V>& q, uint64_t count, const uint32_t* v1, const uint32_t* v2,
                    double* dist, cudaStream_t s) {
    const uint32_t k = q.k;
    // dense grouping: a counting sort over all k^2 pair bins; sparse (batches
    // far smaller than k^2): radix sort of the batch's keys and its runs as
    // the bins, so the cost follows the batch instead of k^2
    const char* ge = std::getenv("PSP_GROUPING");  // dense|sparse override (tests)
    bool sparse = uint64_t(k) * k >= SPARSE_GROUPING_MIN_BINS &&
                  uint64_t(count) * SPARSE_GROUPING_RATIO < uint64_t(k) * k;
    if (ge && std::strcmp(ge, "dense") == 0) sparse = false;
    if (ge && std::strcmp(ge, "sparse") == 0) sparse = true;
    const uint32_t nbins = sparse ? uint32_t(count) : k * k;
    if (!gw.done) CK(cudaEventCreateWithFlags(&gw.done, cudaEventDisableTiming));
    // the workspace is shared by all calls on this oracle: order after the
    // previous user, whatever stream it ran on
    CK(cudaStreamWaitEvent(s, gw.done, 0));
    // u32 arrays of `count` in gw.buf: key l1 l2 best sorted s_l1 s_l2 |
    // sparse: idx key_sorted idx_sorted run_key | 16-bit product: lb fb_list
    // base16 | num_runs, fb_count
    const uint64_t per = 14;
    if (gw.count < count || gw.buf.bytes < (per * count + 4) * sizeof(uint32_t)) {
        CK(cudaStreamSynchronize(s));
        gw.count = std::max<uint64_t>(gw.count, count);
        gw.buf.alloc((per * gw.count + 4) * sizeof(uint32_t));
    }
    if (gw.bins.bytes < size_t(nbins + 1) * 4 * sizeof(uint32_t)) {
        CK(cudaStreamSynchronize(s));
        gw.bins.alloc(size_t(nbins + 1) * 4 * sizeof(uint32_t));
    }
    uint32_t key_bits = 1;
    while (key_bits < 32 && (uint64_t(1) << key_bits) < uint64_t(k) * k) ++key_bits;
    {
        size_t t1 = 0, t2 = 0, t3 = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, t1, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                         int(nbins + 1), s));
        if (sparse) {
            CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                               (uint32_t*)nullptr, (uint32_t*)nullptr, int(count), 0,
                                               int(key_bits), s));
            CK(cub::DeviceRunLengthEncode::Encode(nullptr, t3, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                                  (uint32_t*)nullptr, (uint32_t*)nullptr, int(count), s));
        }
        const size_t need = std::max({t1, t2, t3});
        if (gw.temp.bytes < need) {
            CK(cudaStreamSynchronize(s));
            gw.temp.alloc(need);
        }
        gw.temp_bytes = gw.temp.bytes;
    }
    GroupWork w;
    uint32_t* base = gw.buf.as<uint32_t>();
    const uint64_t C = count;  // layout of this batch (the buffer holds >= per * count)
    w.key = base;
    w.l1 = base + C;
    w.l2 = base + 2 * C;
    w.best = base + 3 * C;
    w.sorted = base + 4 * C;
    w.s_l1 = base + 5 * C;
    w.s_l2 = base + 6 * C;
    w.idx = sparse ? base + 7 * C : nullptr;
    uint32_t* key_sorted = base + 8 * C;
    uint32_t* idx_sorted = base + 9 * C;
    uint32_t* run_key = sparse ? base + 10 * C : nullptr;
    constexpr bool U16 = MODE == QM_BLOCKS16;
    w.lb = U16 ? base + 11 * C : nullptr;
    w.fb_list = U16 ? base + 12 * C : nullptr;
    w.base16 = U16 ? base + 13 * C : nullptr;
    uint32_t* num_runs = base + 14 * C;
    w.fb_count = base + 14 * C + 1;
    w.bin_key = run_key;
    uint32_t* bins = gw.bins.as<uint32_t>();
    w.bin_cnt = bins;
    w.bin_start = bins + (nbins + 1);
    w.task_cnt = bins + 2 * size_t(nbins + 1);
    w.task_start = bins + 3 * size_t(nbins + 1);
    w.nbins = nbins;
    CK(cudaMemsetAsync(w.bin_cnt, 0, size_t(nbins + 1) * sizeof(uint32_t), s));
    const unsigned qb = unsigned((count + 255) / 256);
    group_prep<V, MODE == QM_ROUTED><<<qb, 256, 0, s>>>(q, v1, v2, count, w);
    CK_LAUNCH();
    size_t tb = gw.temp_bytes;
    if (sparse) {
        CK(cub::DeviceRadixSort::SortPairs(gw.temp.p, tb, w.key, key_sorted, w.idx, idx_sorted,
                                           int(count), 0, int(key_bits), s));
        tb = gw.temp_bytes;
        CK(cub::DeviceRunLengthEncode::Encode(gw.temp.p, tb, key_sorted, run_key, w.bin_cnt,
                                              num_runs, int(count), s));
    }
    group_tasks<<<(nbins + 1 + 255) / 256, 256, 0, s>>>(w, q.bnd_off, q.k);
    CK_LAUNCH();
    tb = gw.temp_bytes;
    CK(cub::DeviceScan::ExclusiveSum(gw.temp.p, tb, w.bin_cnt, w.bin_start, int(nbins + 1), s));
    tb = gw.temp_bytes;
    CK(cub::DeviceScan::ExclusiveSum(gw.temp.p, tb, w.task_cnt, w.task_start, int(nbins + 1), s));
    // task records: upper bound on the task count without a host round trip
    {
        uint64_t max_tasks = 0;
        for (uint32_t c = 0; c < k; ++c)
            max_tasks = std::max<uint64_t>(max_tasks, (bnd_off[c + 1] - bnd_off[c] + 31) / 32);
        max_tasks *= (count + GQ - 1) / GQ + std::min<uint64_t>(count, nbins);
        if (gw.tasks.bytes < max_tasks * sizeof(uint4) + 16) {
            CK(cudaStreamSynchronize(s));
            gw.tasks.alloc(max_tasks * sizeof(uint4) + 16);
        }
    }
    w.tasks = gw.tasks.as<uint4>();
    group_emit<<<(nbins + 255) / 256, 256, 0, s>>>(w, q.bnd_off, q.k, MODE == QM_BLOCKS);
    CK_LAUNCH();
    if (sparse) {
        group_scatter_sorted<<<qb, 256, 0, s>>>(count, idx_sorted, w);
    } else {
        CK(cudaMemsetAsync(w.bin_cnt, 0, size_t(nbins) * sizeof(uint32_t), s));
        group_scatter<<<qb, 256, 0, s>>>(count, w);
    }
    CK_LAUNCH();
    const int gsmem = GWARPS * sizeof(WarpStage<V>);
    static bool attr_set = false;  // one flag per <V, MODE> instantiation
    if (!attr_set) {
        CK(cudaFuncSetAttribute(query_grouped<V, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                gsmem));
        attr_set = true;
    }
    if constexpr (U16) {
        CK(cudaMemsetAsync(w.fb_count, 0, sizeof(uint32_t), s));
        group_bases16<V><<<unsigned(std::min<uint64_t>((count + 7) / 8, uint64_t(sms) * 64)), 256, 0, s>>>(
            q, count, w);
        CK_LAUNCH();
    }
    query_grouped<V, MODE><<<sms * 2, GTHREADS, gsmem, s>>>(q, w);
    CK_LAUNCH();
    if constexpr (U16) {
        group_finish16<V><<<qb, 256, 0, s>>>(q, count, w, dist);
        CK_LAUNCH();
        query_fallback<V><<<sms * 2, 32 * QC_WARPS, 0, s>>>(q, v1, v2, w, dist);
        CK_LAUNCH();
        if (std::getenv("PSP_QUERY_STATS")) {  // diagnostics: how many went to the u32 fallback
            uint32_t fb = 0;
            CK(cudaMemcpyAsync(&fb, w.fb_count, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::fprintf(stderr, "[psp] 16-bit product: %u of %llu queries to the u32 fallback\n", fb,
                         (unsigned long long)count);
        }
    } else {
        group_finish<V><<<qb, 256, 0, s>>>(q, v1, v2, count, w, dist);
        CK_LAUNCH();
    }
    CK(cudaEventRecord(gw.done, s));
}

// Kernel choice by batch density (queries per component pair c1 <= c2):
// the pair-grouped kernel reuses each B1 x B2 block from shared memory but
// pays a counting sort over k^2 bins per batch; for batches much smaller than
// that (no reuse to gain) query_cta answers each query with one CTA and no
// sort. query_warp remains for k*k beyond 32-bit bin keys and as the
// PSP_QUERY_KERNEL=warp check. All kernels return identical distances.
// CTA_MAX_DENSITY: measured crossover (profiles/bench/r2_query_kernel_sweep).
constexpr double GROUP_MIN_DENSITY = 0.0;
constexpr double CTA_MAX_DENSITY = 0.0;
// small batches: one launch, no sort (measured on cfg3, block layout, 16-warp
// query_cta: 44.3 vs query_grouped 11.8 M queries/s at 1K pairs, 50.4 vs 47.5
// at 10K, 55.4 vs 62.6 at 30K; profiles/r2/query_cta_shapes_cfg3.jsonl,
// profiles/r2/query_sweep_cfg3_cta_blocks.jsonl)
constexpr uint64_t CTA_MAX_COUNT = 16384;

template <class V>
QueryView<V> query_view(const psp_gpu_oracle* o, uint32_t* bad_id) {
    QueryView<V> q{};
    q.n = static_cast<uint32_t>(o->R.n);
    q.bad_id = bad_id;
    q.perm = o->d_perm.as<uint32_t>();
    q.assign = o->d_assign.as<uint32_t>();
    q.comp_off = o->d_comp_off.as<uint32_t>();
    q.bnd_off = o->d_bnd_off.as<uint32_t>();
    q.cb_off = o->d_cb_off.as<uint64_t>();
    q.cb = o->d_cb.as<V>();
    q.comps = o->comps.view<V>();
    q.bg = o->bg.tiles.as<V>();
    q.bg_nb = o->bg.nmat ? o->bg.nb[0] : 0;
    q.k = o->R.k;
    q.scale = o->scale;
    q.bq = o->bq.p ? o->bq.as<V>() : nullptr;
    q.bq_off = o->bq.p ? o->d_bq_off.as<uint64_t>() : nullptr;
    q.bq16 = o->bq16.p ? o->bq16.as<uint16_t>() : nullptr;
    q.bq16_off = o->bq16.p ? o->d_bq16_off.as<uint64_t>() : nullptr;
    q.bqaux = o->bq16.p ? o->bqaux.as<uint32_t>() : nullptr;
    q.aux_off = o->bq16.p ? o->d_aux_off.as<uint64_t>() : nullptr;
    q.cb16 = o->bq16.p ? o->cb16.as<uint16_t>() : nullptr;
    q.cb16_off = o->bq16.p ? o->d_cb16_off.as<uint64_t>() : nullptr;
    q.rbase = o->bq16.p ? o->d_rbase.as<uint32_t>() : nullptr;
    q.u16_sat = o->u16_sat;
    return q;
}

template <class V>
void launch_queries(const psp_gpu_oracle* o, uint64_t count, const uint32_t* v1,
                    const uint32_t* v2, double* dist, cudaStream_t s, uint32_t* bad_id) {
    if (count == 0) return;
    const QueryView<V> q = query_view<V>(o, bad_id);
    const uint64_t k = o->R.k;
    const double pairs = double(k) * double(k + 1) / 2.0;
    // PSP_QUERY_KERNEL=warp|grouped overrides the density heuristic (tests,
    // profiling); both kernels return identical distances.
    const char* force = std::getenv("PSP_QUERY_KERNEL");
    bool grouped = double(count) >= GROUP_MIN_DENSITY * pairs;
    bool cta = double(count) < CTA_MAX_DENSITY * pairs || count <= CTA_MAX_COUNT;
    if (force && std::strcmp(force, "warp") == 0) grouped = cta = false;
    if (force && std::strcmp(force, "grouped") == 0) grouped = true, cta = false;
    if (force && std::strcmp(force, "cta") == 0) cta = true;
    if (cta) {
        const unsigned blocks = unsigned(std::min<uint64_t>(count, uint64_t(o->ctx->sms) * 8));
        query_cta<V, QC_BATCH_WARPS, 4, QC_BATCH_MINB><<<blocks, 32 * QC_BATCH_WARPS, 0, s>>>(
            q, v1, v2, count, dist);
        CK_LAUNCH();
        return;
    }
    if (grouped && k * k < (1ull << 31) && count < (1ull << 31)) {
        // (callers hold o->query_mu: the workspace map and its growth)
        GroupWorkspace& ws = const_cast<psp_gpu_oracle*>(o)->workspace_for(s);
        // the block query layout when it was built (PSP_QUERY_LAYOUT=tiles
        // forces the tile-packed path; both give identical distances)
        const char* lay = std::getenv("PSP_QUERY_LAYOUT");
        const char* prod = std::getenv("PSP_QUERY_PRODUCT");
        const bool lane_product = prod && std::strcmp(prod, "lane") == 0;
        const bool p8x8 = prod && std::strcmp(prod, "8x8") == 0;
        const char* u16env = std::getenv("PSP_QUERY_U16");
        const bool u16 = q.bq16 && !(lay && std::strcmp(lay, "tiles") == 0) && !lane_product &&
                         !p8x8 && u16env && std::strcmp(u16env, "1") == 0;
        if constexpr (std::is_same<V, uint32_t>::value) {
            if (u16) {
                launch_grouped<V, QM_BLOCKS16>(ws, o->R.bnd_off, o->ctx->sms, q, count, v1, v2, dist, s);
                return;
            }
        }
        if (q.bq && !(lay && std::strcmp(lay, "tiles") == 0) && lane_product)
            launch_grouped<V, QM_BLOCKS_LANE>(ws, o->R.bnd_off,
                                              o->ctx->sms, q, count, v1, v2, dist, s);
        else if (q.bq && !(lay && std::strcmp(lay, "tiles") == 0) && p8x8)
            launch_grouped<V, QM_BLOCKS_8X8>(ws, o->R.bnd_off,
                                             o->ctx->sms, q, count, v1, v2, dist, s);
        else if (q.bq && !(lay && std::strcmp(lay, "tiles") == 0))
            launch_grouped<V, QM_BLOCKS>(ws, o->R.bnd_off,
                                         o->ctx->sms, q, count, v1, v2, dist, s);
        else
            launch_grouped<V, QM_TILES>(ws, o->R.bnd_off,
                                        o->ctx->sms, q, count, v1, v2, dist, s);
        return;
    }
    const uint64_t warps_per_block = 8;
    const uint64_t want = (count + warps_per_block - 1) / warps_per_block;
    const unsigned blocks =
        unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(o->ctx->sms) * 16)));
    query_warp<V><<<blocks, 256, 0, s>>>(q, v1, v2, count, dist);
    CK_LAUNCH();
}

// Point queries (count <= MAILBOX_PAIRS) through the resident server CTA:
// no launch and no stream sync per call while the server is up (it idles out
// after PSP_SERVER_IDLE_US, default 200 us). Caller holds o->query_mu.
template <class V>
bool point_queries(psp_gpu_oracle* o, uint64_t count, const uint32_t* v1, const uint32_t* v2,
                   double* dist) {
    if (count == 0 || count > uint64_t(MAILBOX_PAIRS)) return false;
    if (std::getenv("PSP_NO_QUERY_SERVER")) return false;
    if (!o->mb) {
        void* p = nullptr;
        CK(cudaHostAlloc(&p, sizeof(QueryMailbox), cudaHostAllocMapped | cudaHostAllocPortable));
        std::memset(p, 0, sizeof(QueryMailbox));
        o->mb = static_cast<QueryMailbox*>(p);
        CK(cudaStreamCreateWithFlags(&o->srv, cudaStreamNonBlocking));
    }
    const char* idle_env = std::getenv("PSP_SERVER_IDLE_US");
    const unsigned long long idle_ns =
        (idle_env ? std::strtoull(idle_env, nullptr, 10) : 200ull) * 1000ull;
    QueryMailbox* mb = o->mb;
    // 16-bit request tags; 0 is the initial (never requested) state
    uint32_t seq = uint32_t(++o->srv_seq) & 0xffffu;
    if (seq == 0) seq = uint32_t(++o->srv_seq) & 0xffffu;
    const unsigned long long tag = (unsigned long long)seq << 48;
    auto launch = [&] {
        mb->alive = 1u;  // until the kernel says otherwise
        const size_t smem = server_smem_bytes(o->R.n, o->R.k);
        static bool attr_set = false;  // one per V (callers hold query_mu of some oracle)
        static std::mutex attr_mu;
        {
            std::lock_guard<std::mutex> lk(attr_mu);
            if (!attr_set) {
                CK(cudaFuncSetAttribute(query_server<V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        192 << 10));
                attr_set = true;
            }
        }
        // `last` = any tag but this request's: the pending request is served
        query_server<V><<<1, 32 * QC_WARPS, smem, o->srv>>>(query_view<V>(o, nullptr), mb,
                                                            seq ^ 0x8000u, idle_ns, smem ? 1 : 0);
        CK_LAUNCH();
    };
    // every word carries the request tag: the order of the stores is free
    // (the first line last, so a single poll usually sees a whole request)
    for (uint64_t i = 1; i < count; ++i) {
        mb->req[2 * i] = tag | v1[i];
        mb->req[2 * i + 1] = tag | v2[i];
    }
    static const bool prof = std::getenv("PSP_SERVER_PROFILE") != nullptr;
    const auto tp = prof ? Clock::now() : Clock::time_point{};
    mb->req[1] = tag | v2[0];
    mb->req[0] = tag | (uint64_t(count) << 32) | v1[0];
    std::atomic_thread_fence(std::memory_order_seq_cst);
    if (!mb->alive && cudaStreamQuery(o->srv) == cudaSuccess) launch();
    const auto t0 = Clock::now();
    const uint64_t last_word = 2 * count;  // the bad flag, written with the rest
    for (uint64_t spin = 1;; ++spin) {
        bool done = true;
        for (uint64_t w = 0; w <= last_word && done; ++w) done = mb_tag(mb->ans[w]) == seq;
        if (done) break;
        if ((spin & 255) == 0 && !mb->alive) {
            // the server idled out (possibly racing this request): once its
            // kernel is gone, start another unless the answer arrived
            const cudaError_t e = cudaStreamQuery(o->srv);
            if (e == cudaSuccess) {
                bool arrived = true;
                for (uint64_t w = 0; w <= last_word && arrived; ++w)
                    arrived = mb_tag(mb->ans[w]) == seq;
                if (!arrived) launch();
            } else if (e != cudaErrorNotReady) {
                CK(e);
            }
        }
        if ((spin & 0xfffff) == 0 && ms_since(t0) > 60000.0)
            throw Fail{PSP_ECUDA, "point-query server did not answer within 60 s"};
    }
    if (prof) {
        o->srv_prof[0] += 1;
        o->srv_prof[1] += std::chrono::duration<double, std::nano>(Clock::now() - tp).count();
        o->srv_prof[2] += double(mb->prof[1] - mb->prof[0]);
    }
    const bool bad = uint32_t(mb->ans[last_word]) != 0;
    for (uint64_t i = 0; i < count; ++i) {
        const unsigned long long bits = (mb->ans[2 * i] & 0xffffffffull) |
                                        ((mb->ans[2 * i + 1] & 0xffffffffull) << 32);
        std::memcpy(&dist[i], &bits, sizeof(double));
    }
    if (bad) throw ArgError("query: vertex id out of range");  // src/query.cpp:30
    return true;
}

}  // namespace


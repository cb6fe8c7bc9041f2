// engine_shard.cuh — routed (sharded) queries: the paper's distributed query
// mode (src/cluster.cpp routed_query :66-92, ClusterSim::execute :169-206)
// on real GPUs instead of simulated workers.
//
// Placement (src/placement.cpp:7-33) gives every component one owner rank.
// Rank r keeps only what its components need:
//   * the full boundary rows BT[c] (|B(C)| x b) of every owned c, dense and
//     row-major, built from the replicated symmetric boundary table;
//   * the to-boundary rows CT[c][l][0..|B(C)|) of owned c (a compact arena);
//   * the full component tables of owned c (the same-component cap).
// A query (v1, v2) executes at owner(C1) like the reference's: its ids are
// sent there (NCCL send/recv), stitched against BT[C1] with row1 from the
// local arena, and combined with col2 = CT[C2][l2][..], which query_grouped
// reads straight out of owner(C2)'s arena over NVLink when the owners differ
// (CUDA IPC mapping; the paper's Alg. 2 line 8 transfer, B2 entries). The
// distance returns to the caller's rank and order.
//
// Transfer accounting is the reference's: a query whose two components have
// different owners moves B2 entries, 8 bytes each (cluster.cpp:81-84); the
// per-query executed_on / column_owner / transfer_entries are returned so the
// host can keep the TransferLedger.
#pragma once

struct psp_gpu_shard {
    psp_gpu_ctx* ctx = nullptr;
    Kind kind{PSP_VALUE_U32, 0};
    double scale = 1.0;
    uint64_t n = 0, b = 0;
    uint32_t k = 0;
    std::vector<uint32_t> owner, bnd_off;
    DBuf d_perm, d_assign, d_comp_off, d_bnd_off, d_owner, d_cb_off, d_cb, d_cb_peer;
    DBuf d_bt, d_bt_row0;
    uint64_t bt_stride = 0, bt_rows = 0;
    MatArena comps;  // owned components only (the others have size 0)
    std::vector<void*> opened;  // peer arenas mapped through CUDA IPC
    GroupWorkspace gw;
    DBuf stage, recv, out, gath;  // routing buffers (grow-only, reused per batch)
    std::mutex mu;   // one routed batch at a time (the batch is collective)
    uint64_t device_bytes = 0;
    ~psp_gpu_shard() {
        for (void* p : opened) cudaIpcCloseMemHandle(p);
    }
};

namespace {

template <class V>
__global__ void gather_bt_rows(const V* __restrict__ bg, uint32_t nb, uint64_t b,
                               const uint32_t* __restrict__ row_gid, uint64_t nrows,
                               uint64_t stride, V* __restrict__ bt) {
    const uint64_t total = nrows * stride;
    for (uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = idx / stride, j = idx - r * stride;
        bt[idx] = j < b ? bg[sym_off(row_gid[r], static_cast<uint32_t>(j), nb)] : Ops<V>::inf();
    }
}

// Row-sharded storage (psp_gpu_oracle::row_storage): rows `row_gid`
// (boundary ids) of the full table as far as this rank holds them -- element
// (p, q) of the K2 working matrix lives in tile row min(p, q) / T, owned by
// rank (that row mod world) -- and INF elsewhere. The destination rank
// min-reduces every rank's part (ncclReduce), so each element arrives from
// exactly the rank that holds it. grid: (column blocks, rows).
template <class V>
__global__ void gather_bt_part(const V* __restrict__ W, uint32_t nbW, const uint32_t* __restrict__ pos,
                               uint32_t rank, uint32_t world, uint64_t b,
                               const uint32_t* __restrict__ row_gid, uint64_t stride,
                               V* __restrict__ out) {
    const uint64_t r = blockIdx.y;
    const uint32_t p = pos[row_gid[r]];
    V* dst = out + r * stride;
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < stride;
         j += uint64_t(gridDim.x) * blockDim.x) {
        V v = Ops<V>::inf();
        if (j < b) {
            const uint32_t q = pos[j];
            if ((min(p, q) / T) % world == rank) v = W[sym_off(p, q, nbW)];
        }
        dst[j] = v;
    }
}

struct RouteView {
    const uint32_t* perm;
    const uint32_t* assign;
    const uint32_t* bnd_off;
    const uint32_t* owner;
    uint32_t n, world;
};

// Per query: validate ids, executing rank = owner(C1), and the reference's
// routing facts (cluster.cpp:77-85). counts[r] = queries bound for rank r;
// totals = {transfer queries, transfer entries}.
__global__ void route_prep(RouteView rv, const uint32_t* __restrict__ v1,
                           const uint32_t* __restrict__ v2, uint64_t count,
                           uint32_t* __restrict__ exec, uint32_t* __restrict__ counts,
                           uint32_t* __restrict__ bad, unsigned long long* __restrict__ totals,
                           uint32_t* __restrict__ out_exec, uint32_t* __restrict__ out_col,
                           uint32_t* __restrict__ out_entries) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint32_t a = v1[i], c = v2[i];
    if (a >= rv.n || c >= rv.n) {  // src/query.cpp:30
        *bad = 1u;
        a = c = 0;
    }
    const uint32_t c1 = rv.assign[rv.perm[a]], c2 = rv.assign[rv.perm[c]];
    const uint32_t e = rv.owner[c1], co = rv.owner[c2];
    const uint32_t b2 = rv.bnd_off[c2 + 1] - rv.bnd_off[c2];
    exec[i] = e;
    atomicAdd(&counts[e], 1u);
    if (e != co) {
        atomicAdd(&totals[0], 1ull);
        atomicAdd(&totals[1], (unsigned long long)b2);
    }
    out_exec[i] = e;
    out_col[i] = co;
    out_entries[i] = e != co ? b2 : 0u;
}

// Bucket the queries by executing rank: slot[i] = its position in the send
// buffers (rank-major; order inside a bucket is whatever the atomics give,
// the answers come back through slot[]).
__global__ void route_scatter(const uint32_t* __restrict__ v1, const uint32_t* __restrict__ v2,
                              uint64_t count, const uint32_t* __restrict__ exec,
                              const uint32_t* __restrict__ send_off, uint32_t* __restrict__ cursor,
                              uint32_t* __restrict__ slot, uint32_t* __restrict__ s1,
                              uint32_t* __restrict__ s2) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t e = exec[i];
    const uint32_t at = send_off[e] + atomicAdd(&cursor[e], 1u);
    slot[i] = at;
    s1[at] = v1[i];
    s2[at] = v2[i];
}

__global__ void route_gather(const double* __restrict__ back, const uint32_t* __restrict__ slot,
                             uint64_t count, double* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) out[i] = back[slot[i]];
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Fail{PSP_ENCCL, std::string(what) + ": " + pspg::nccl().GetErrorString(r)};
}

// Component placement (src/placement.cpp:7-33).
std::vector<uint32_t> place(uint32_t k, uint32_t p, int policy) {
    if (p < 1) throw ArgError("place_components: need at least one worker");
    if (p > k) throw ArgError("place_components: more workers than components");
    std::vector<uint32_t> owner(k);
    if (policy == PSP_PLACE_ROUND_ROBIN) {
        for (uint32_t c = 0; c < k; ++c) owner[c] = c % p;
    } else if (policy == PSP_PLACE_PAIRS_PER_GPU) {
        const uint32_t base = k / p, extra = k % p;
        uint32_t c = 0;
        for (uint32_t w = 0; w < p; ++w)
            for (uint32_t i = 0; i < base + (w < extra ? 1u : 0u); ++i) owner[c++] = w;
    } else {
        throw ArgError("place_components: unknown placement policy");
    }
    return owner;
}

template <class V>
void shard_build(psp_gpu_shard* sh, const psp_gpu_oracle* o) {
    psp_gpu_ctx* ctx = sh->ctx;
    cudaStream_t s = ctx->stream;
    const Reordered& R = o->R;
    const uint32_t k = R.k, me = static_cast<uint32_t>(ctx->rank);
    const size_t vb = sizeof(V);
    const auto t0 = Clock::now();
    auto lap = [&](const char* what) {  // PSP_FW_PROFILE: synchronised laps
        if (!std::getenv("PSP_FW_PROFILE")) return;
        CK(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[psp] rank %d shard lap: %s at %.1f ms\n", ctx->rank, what, ms_since(t0));
    };
    auto d2d = [&](DBuf& dst, const DBuf& src) {
        dst.alloc(src.bytes);
        CK(cudaMemcpyAsync(dst.p, src.p, src.bytes, cudaMemcpyDeviceToDevice, s));
    };
    d2d(sh->d_perm, o->d_perm);
    d2d(sh->d_assign, o->d_assign);
    d2d(sh->d_comp_off, o->d_comp_off);
    d2d(sh->d_bnd_off, o->d_bnd_off);
    sh->d_owner = upload(sh->owner, s);

    // compact to-boundary arenas: c sits at cb_off[c] in owner(c)'s arena
    std::vector<uint64_t> src_off(k + 1, 0), cb_off(k, 0), used(ctx->world, 0);
    for (uint32_t c = 0; c < k; ++c) {
        const uint64_t sz = uint64_t(R.comp_off[c + 1] - R.comp_off[c]) *
                            cb_stride(R.bnd_off[c + 1] - R.bnd_off[c]);
        src_off[c + 1] = src_off[c] + sz;
        cb_off[c] = used[sh->owner[c]];
        used[sh->owner[c]] += sz;
    }
    sh->d_cb.alloc_ipc(used[me] * vb);  // mapped into the peers (CUDA IPC)
    for (uint32_t c = 0; c < k; ++c)
        if (sh->owner[c] == me && src_off[c + 1] > src_off[c])
            CK(cudaMemcpyAsync(sh->d_cb.as<V>() + cb_off[c], o->d_cb.as<V>() + src_off[c],
                               (src_off[c + 1] - src_off[c]) * vb, cudaMemcpyDeviceToDevice, s));
    sh->d_cb_off = upload(cb_off, s);
    lap("to-boundary rows");

    // dense full boundary rows of the owned components
    sh->bt_stride = std::max<uint64_t>(4, (sh->b + 3) & ~uint64_t(3));
    std::vector<uint32_t> row0(k, 0), gid;
    for (uint32_t c = 0; c < k; ++c) {
        if (sh->owner[c] != me) continue;
        row0[c] = static_cast<uint32_t>(gid.size());
        for (uint32_t t = R.bnd_off[c]; t < R.bnd_off[c + 1]; ++t) gid.push_back(t);
    }
    sh->bt_rows = gid.size();
    sh->d_bt_row0 = upload(row0, s);
    sh->d_bt.alloc(sh->bt_rows * sh->bt_stride * vb);
    lap("boundary rows allocated");
    if (o->row_storage) {
        // the table is spread over the ranks by tile row: every rank sends
        // its part of each destination's rows, min-reduced at the destination
        // (rank order, destination rows in chunks of <= 256 MB)
        auto& api = pspg::nccl();
        const uint64_t row_bytes = sh->bt_stride * vb;
        const uint64_t per = std::max<uint64_t>(1, std::min<uint64_t>(65535, (256ull << 20) / row_bytes));
        std::vector<uint32_t> all_gid;
        std::vector<uint64_t> dst_off(ctx->world + 1, 0);
        for (int d = 0; d < ctx->world; ++d) {
            for (uint32_t c = 0; c < k; ++c)
                if (sh->owner[c] == uint32_t(d))
                    for (uint32_t t = R.bnd_off[c]; t < R.bnd_off[c + 1]; ++t) all_gid.push_back(t);
            dst_off[d + 1] = all_gid.size();
        }
        DBuf d_all = upload(all_gid, s);
        DBuf stage(std::min<uint64_t>(per, std::max<uint64_t>(1, all_gid.size())) * row_bytes);
        const ncclDataType_t dt = std::is_same<V, float>::value ? ncclFloat32 : ncclUint32;
        const unsigned gx = unsigned(std::min<uint64_t>(8, (sh->bt_stride + 1023) / 1024));
        for (int d = 0; d < ctx->world; ++d) {
            for (uint64_t r0 = dst_off[d]; r0 < dst_off[d + 1]; r0 += per) {
                const uint64_t nr = std::min<uint64_t>(per, dst_off[d + 1] - r0);
                gather_bt_part<V><<<dim3(gx, unsigned(nr)), 1024, 0, s>>>(
                    o->bg.tiles_as<V>(), o->bg.nb[0], o->d_bg_pos.as<uint32_t>(), me,
                    uint32_t(ctx->world), sh->b, d_all.as<uint32_t>() + r0, sh->bt_stride,
                    stage.as<V>());
                CK_LAUNCH();
                V* recv = d == int(me) ? sh->d_bt.as<V>() + (r0 - dst_off[d]) * sh->bt_stride : stage.as<V>();
                nccl_check(api.Reduce(stage.p, recv, nr * sh->bt_stride, dt, ncclMin, d, ctx->comm, s),
                           "ncclReduce(boundary rows)");
            }
        }
        CK(cudaStreamSynchronize(s));  // d_all and stage die here
    } else if (sh->bt_rows && o->bg.nmat) {
        DBuf d_gid = upload(gid, s);
        gather_bt_rows<V><<<ctx->sms * 8, 256, 0, s>>>(o->bg.tiles_as<V>(), o->bg.nb[0], sh->b,
                                                       d_gid.as<uint32_t>(), sh->bt_rows,
                                                       sh->bt_stride, sh->d_bt.as<V>());
        CK_LAUNCH();
        CK(cudaStreamSynchronize(s));  // d_gid is freed on return
    }

    lap("boundary rows gathered");
    // full component tables of the owned components (same-component cap)
    std::vector<uint64_t> sizes(k, 0);
    for (uint32_t c = 0; c < k; ++c)
        if (sh->owner[c] == me) sizes[c] = R.comp_off[c + 1] - R.comp_off[c];
    sh->comps.create(sizes, vb, false, s);
    for (uint32_t c = 0; c < k; ++c) {
        if (sh->owner[c] != me || sizes[c] == 0) continue;
        const uint64_t elems = ntiles_upper(sh->comps.nb[c]) * TT;
        CK(cudaMemcpyAsync(sh->comps.tiles.as<V>() + sh->comps.tile_base[c],
                           o->comps.tiles.as<V>() + o->comps.tile_base[c], elems * vb,
                           cudaMemcpyDeviceToDevice, s));
    }

    // every rank's arena base: its own, and the peers' mapped over NVLink
    std::vector<uint64_t> bases(ctx->world, 0);
    bases[me] = reinterpret_cast<uint64_t>(sh->d_cb.p);
    if (ctx->world > 1) {
        auto& api = pspg::nccl();
        cudaIpcMemHandle_t mine;
        CK(cudaIpcGetMemHandle(&mine, sh->d_cb.p));
        const size_t hb = sizeof(cudaIpcMemHandle_t);
        DBuf all(hb * ctx->world);
        CK(cudaMemcpyAsync(all.as<char>() + hb * me, &mine, hb, cudaMemcpyHostToDevice, s));
        nccl_check(api.AllGather(all.as<char>() + hb * me, all.p, hb, ncclUint8, ctx->comm, s),
                   "ncclAllGather(ipc handles)");
        std::vector<cudaIpcMemHandle_t> h(ctx->world);
        CK(cudaMemcpyAsync(h.data(), all.p, hb * ctx->world, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int r = 0; r < ctx->world; ++r) {
            if (uint32_t(r) == me) continue;
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, h[r], cudaIpcMemLazyEnablePeerAccess));
            sh->opened.push_back(p);
            bases[r] = reinterpret_cast<uint64_t>(p);
        }
    }
    lap("component tables + peer mapping");
    sh->d_cb_peer = upload(bases, s);
    if (ctx->world > 1) {
        // open the point-to-point channels now: NCCL connects send/recv
        // peers lazily, which would otherwise land in the first batch
        auto& api = pspg::nccl();
        DBuf tiny(2 * 4 * ctx->world);
        CK(cudaMemsetAsync(tiny.p, 0, tiny.bytes, s));
        nccl_check(api.GroupStart(), "ncclGroupStart");
        for (int r = 0; r < ctx->world; ++r) {
            nccl_check(api.Send(tiny.as<uint32_t>() + r, 1, ncclUint32, r, ctx->comm, s), "ncclSend");
            nccl_check(api.Recv(tiny.as<uint32_t>() + ctx->world + r, 1, ncclUint32, r, ctx->comm, s),
                       "ncclRecv");
        }
        nccl_check(api.GroupEnd(), "ncclGroupEnd");
    }
    CK(cudaStreamSynchronize(s));
    lap("NCCL send/recv channels connected");
    sh->device_bytes = sh->d_cb.bytes + sh->d_bt.bytes + sh->comps.bytes() + sh->d_perm.bytes +
                       sh->d_assign.bytes;
}

template <class V>
QueryView<V> shard_view(const psp_gpu_shard* sh) {
    QueryView<V> q{};
    q.perm = sh->d_perm.as<uint32_t>();
    q.assign = sh->d_assign.as<uint32_t>();
    q.comp_off = sh->d_comp_off.as<uint32_t>();
    q.bnd_off = sh->d_bnd_off.as<uint32_t>();
    q.cb_off = sh->d_cb_off.as<uint64_t>();
    q.cb = sh->d_cb.as<V>();
    q.comps = sh->comps.view<V>();
    q.bg = nullptr;
    q.bg_nb = 0;
    q.k = sh->k;
    q.n = static_cast<uint32_t>(sh->n);
    q.bad_id = nullptr;
    q.scale = sh->scale;
    q.bt = sh->d_bt.as<V>();
    q.bt_stride = sh->bt_stride;
    q.bt_row0 = sh->d_bt_row0.as<uint32_t>();
    q.owner = sh->d_owner.as<uint32_t>();
    q.cb_peer = sh->d_cb_peer.as<const V*>();
    return q;
}

// The collective batch: every rank passes its own pairs (possibly none).
template <class V>
void routed_batch(psp_gpu_shard* sh, uint64_t count, const uint32_t* v1, const uint32_t* v2,
                  double* dist, uint32_t* exec_on, uint32_t* col_owner, uint32_t* entries,
                  psp_routed_stats* st) {
    psp_gpu_ctx* ctx = sh->ctx;
    cudaStream_t s = ctx->stream;
    const uint32_t world = static_cast<uint32_t>(ctx->world), me = static_cast<uint32_t>(ctx->rank);
    auto& api = pspg::nccl();
    // staging: v1 v2 exec slot outE outC outN s1 s2 (u32 x count), back (f64
    // x count), counts[world + 1] + cursor[world] + send_off[world], totals
    const uint64_t cnt = std::max<uint64_t>(count, 1);
    const size_t need = cnt * (9 * 4 + 8) + (4 * world + 8) * 4 + 64;
    if (sh->stage.bytes < need) {
        CK(cudaStreamSynchronize(s));
        sh->stage.alloc(need);
    }
    uint32_t* d1 = sh->stage.as<uint32_t>();
    uint32_t* d2 = d1 + cnt;
    uint32_t* dexec = d2 + cnt;
    uint32_t* dslot = dexec + cnt;
    uint32_t* oE = dslot + cnt;
    uint32_t* oC = oE + cnt;
    uint32_t* oN = oC + cnt;
    uint32_t* s1 = oN + cnt;
    uint32_t* s2 = s1 + cnt;
    double* back = reinterpret_cast<double*>(s2 + cnt + (cnt & 1));
    uint32_t* meta = reinterpret_cast<uint32_t*>(back + cnt);
    uint32_t* counts = meta;                 // [world] + bad flag
    uint32_t* cursor = meta + world + 1;     // [world]
    uint32_t* send_off = cursor + world;     // [world]
    unsigned long long* totals =
        reinterpret_cast<unsigned long long*>(meta + ((3 * world + 1 + 1) & ~1u));
    CK(cudaMemsetAsync(meta, 0, (4 * world + 8) * 4, s));
    if (count) {
        CK(cudaMemcpyAsync(d1, v1, count * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d2, v2, count * 4, cudaMemcpyHostToDevice, s));
        RouteView rv{sh->d_perm.as<uint32_t>(), sh->d_assign.as<uint32_t>(),
                     sh->d_bnd_off.as<uint32_t>(), sh->d_owner.as<uint32_t>(),
                     static_cast<uint32_t>(sh->n), world};
        route_prep<<<unsigned((count + 255) / 256), 256, 0, s>>>(rv, d1, d2, count, dexec, counts,
                                                                  counts + world, totals, oE, oC, oN);
        CK_LAUNCH();
    }
    // all ranks learn the full count matrix and every bad-id flag at once,
    // so an invalid id fails the batch on every rank together
    std::vector<uint32_t> all(size_t(world) * (world + 1), 0);
    if (world > 1) {
        if (sh->gath.bytes < all.size() * 4) sh->gath.alloc(all.size() * 4);
        nccl_check(api.AllGather(counts, sh->gath.p, world + 1, ncclUint32, ctx->comm, s),
                   "ncclAllGather(route counts)");
        CK(cudaMemcpyAsync(all.data(), sh->gath.p, all.size() * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    } else {
        CK(cudaMemcpyAsync(all.data(), counts, (world + 1) * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    for (uint32_t r = 0; r < world; ++r)
        if (all[size_t(r) * (world + 1) + world]) throw ArgError("query: vertex id out of range");
    std::vector<uint32_t> soff(world, 0), roff(world + 1, 0), scnt(world), rcnt(world);
    uint64_t acc = 0;
    for (uint32_t r = 0; r < world; ++r) {
        scnt[r] = all[size_t(me) * (world + 1) + r];
        rcnt[r] = all[size_t(r) * (world + 1) + me];
        soff[r] = static_cast<uint32_t>(acc);
        acc += scnt[r];
    }
    for (uint32_t r = 0; r < world; ++r) roff[r + 1] = roff[r] + rcnt[r];
    const uint64_t R = roff[world];
    if (count) {
        CK(cudaMemcpyAsync(send_off, soff.data(), world * 4, cudaMemcpyHostToDevice, s));
        route_scatter<<<unsigned((count + 255) / 256), 256, 0, s>>>(d1, d2, count, dexec, send_off,
                                                                     cursor, dslot, s1, s2);
        CK_LAUNCH();
    }
    // receive side: R pairs to execute here, their answers, all in
    // (origin rank, arrival) order
    uint32_t *r1 = s1, *r2 = s2;
    double *rd = back, *sd = back;
    EventTimer t_route, t_exec;
    t_route.start(s);
    if (world > 1) {
        const uint64_t rc = std::max<uint64_t>(R, 1) + (R & 1);  // keeps rd 8-byte aligned
        if (sh->recv.bytes < rc * 16) {
            CK(cudaStreamSynchronize(s));
            sh->recv.alloc(rc * 16);
        }
        r1 = sh->recv.as<uint32_t>();
        r2 = r1 + rc;
        rd = reinterpret_cast<double*>(r2 + rc);
        nccl_check(api.GroupStart(), "ncclGroupStart");
        for (uint32_t r = 0; r < world; ++r) {
            if (scnt[r]) {
                nccl_check(api.Send(s1 + soff[r], scnt[r], ncclUint32, int(r), ctx->comm, s), "ncclSend");
                nccl_check(api.Send(s2 + soff[r], scnt[r], ncclUint32, int(r), ctx->comm, s), "ncclSend");
            }
            if (rcnt[r]) {
                nccl_check(api.Recv(r1 + roff[r], rcnt[r], ncclUint32, int(r), ctx->comm, s), "ncclRecv");
                nccl_check(api.Recv(r2 + roff[r], rcnt[r], ncclUint32, int(r), ctx->comm, s), "ncclRecv");
            }
        }
        nccl_check(api.GroupEnd(), "ncclGroupEnd");
    }
    t_route.stop(s);
    t_exec.start(s);
    if (R) {
        const QueryView<V> q = shard_view<V>(sh);
        launch_grouped<V, QM_ROUTED>(sh->gw, sh->bnd_off, ctx->sms, q, R, r1, r2, rd, s);
    }
    t_exec.stop(s);
    if (world > 1) {
        nccl_check(api.GroupStart(), "ncclGroupStart");
        for (uint32_t r = 0; r < world; ++r) {
            if (rcnt[r])
                nccl_check(api.Send(rd + roff[r], rcnt[r], ncclFloat64, int(r), ctx->comm, s), "ncclSend");
            if (scnt[r])
                nccl_check(api.Recv(sd + soff[r], scnt[r], ncclFloat64, int(r), ctx->comm, s), "ncclRecv");
        }
        nccl_check(api.GroupEnd(), "ncclGroupEnd");
    }
    unsigned long long tot[2] = {0, 0};
    if (count) {
        // sd holds this rank's answers in send order
        if (sh->out.bytes < count * 8) {
            CK(cudaStreamSynchronize(s));
            sh->out.alloc(count * 8);
        }
        route_gather<<<unsigned((count + 255) / 256), 256, 0, s>>>(sd, dslot, count,
                                                                    sh->out.as<double>());
        CK_LAUNCH();
        CK(cudaMemcpyAsync(dist, sh->out.p, count * 8, cudaMemcpyDeviceToHost, s));
        if (exec_on) CK(cudaMemcpyAsync(exec_on, oE, count * 4, cudaMemcpyDeviceToHost, s));
        if (col_owner) CK(cudaMemcpyAsync(col_owner, oC, count * 4, cudaMemcpyDeviceToHost, s));
        if (entries) CK(cudaMemcpyAsync(entries, oN, count * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(tot, totals, sizeof(tot), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    } else {
        CK(cudaStreamSynchronize(s));
    }
    if (st) {
        st->queries = count;
        st->executed_here = R;
        st->sent_to_peers = count - scnt[me];
        st->transfer_queries = tot[0];
        st->transfer_entries = tot[1];
        st->transfer_bytes = 8 * tot[1];  // f64 accounting, src/cluster.cpp:83
        st->route_ms = t_route.ms();
        st->exec_ms = t_exec.ms();
    }
}

}  // namespace

// psp_gpu.cu — C-ABI (include/psp_gpu.h) over the sm_100a kernels.
//
// Device build pipeline (replaces src/oracle.cpp:144-194 Phases 2 and 3):
//   host   partition_graph + reorder            (identical ids to the reference)
//   K0     component tiles <- INF / 0 diagonal / intra-component edge weights
//   K1     batched symmetric blocked FW over all k component matrices
//   BG     BG tiles <- INF / 0 diagonal / component boundary blocks (clique
//          edges, src/oracle.cpp:110-122) / cross edges (:103-109)
//   K2     symmetric blocked FW on the b x b boundary-graph matrix (replaces
//          one Dijkstra per boundary vertex, :127-142; equal distances)
//   CB     |C| x |B(C)| to-boundary tables for the query kernel
// Queries (K3, src/query.cpp:85-114) read CB, the BG tiles and, for
// same-component pairs, the component tiles.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <type_traits>
#include <string>
#include <vector>

#include "fw_kernels.cuh"
#include "host_graph.hpp"
#include "minplus.cuh"
#include "nccl_api.hpp"
#include "oracle_file.cuh"
#include "psp_gpu.h"
#include "query_kernels.cuh"

using namespace pspg;

namespace {

thread_local std::string g_err;

struct Fail {
    psp_status st;
    std::string msg;
};

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw Fail{e_ == cudaErrorMemoryAllocation ? PSP_ENOMEM : PSP_ECUDA,       \
                       std::string(#x) + ": " + cudaGetErrorString(e_)};               \
    } while (0)
#define CK_LAUNCH(what) CK(cudaGetLastError())

template <typename F>
psp_status guarded(F&& f) {
    try {
        f();
        return PSP_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.st;
    } catch (const GraphError& e) {
        g_err = e.what();
        return PSP_EGRAPH;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return PSP_EINVAL;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return PSP_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PSP_ECUDA;
    }
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
}

// ------------------------------------------------------ device buffers --
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    explicit DBuf(size_t n) { alloc(n); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DBuf() { reset(); }
    void alloc(size_t n) {
        reset();
        if (n == 0) n = 16;
        CK(cudaMalloc(&p, n));
        bytes = n;
    }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

template <class T>
DBuf upload(const std::vector<T>& h, cudaStream_t s) {
    DBuf d(h.size() * sizeof(T));
    if (!h.empty()) CK(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
}

// A batch of symmetric tile-packed matrices (see minplus.cuh).
struct MatArena {
    uint32_t nmat = 0, nb_max = 0;
    size_t vbytes = 4;
    std::vector<uint32_t> nb;
    std::vector<uint64_t> tile_base, panel_base, work_prefix;
    uint64_t tile_elems = 0, panel_elems = 0;
    DBuf tiles, panel, d_tile_base, d_panel_base, d_work_prefix, d_nb;
    // row ownership for the multi-GPU boundary graph (nmat == 1)
    uint32_t rank = 0, world = 1, nrows = 0;
    DBuf d_rows, d_row_prefix;

    void shard_rows(uint32_t r, uint32_t g, cudaStream_t s) {
        rank = r;
        world = g;
        std::vector<uint32_t> rows;
        std::vector<uint64_t> prefix(1, 0);
        for (uint32_t I = r; I < nb[0]; I += g) {
            rows.push_back(I);
            prefix.push_back(prefix.back() + (nb[0] - I));
        }
        nrows = static_cast<uint32_t>(rows.size());
        d_rows = upload(rows, s);
        d_row_prefix = upload(prefix, s);
    }

    void create(const std::vector<uint64_t>& sizes, size_t value_bytes, bool with_panel,
                cudaStream_t s) {
        vbytes = value_bytes;
        nmat = static_cast<uint32_t>(sizes.size());
        nb.resize(nmat);
        tile_base.resize(nmat);
        panel_base.resize(nmat);
        work_prefix.assign(nmat + 1, 0);
        tile_elems = panel_elems = 0;
        nb_max = 0;
        for (uint32_t m = 0; m < nmat; ++m) {
            nb[m] = static_cast<uint32_t>((sizes[m] + T - 1) / T);
            nb_max = std::max(nb_max, nb[m]);
            tile_base[m] = tile_elems;
            panel_base[m] = panel_elems;
            tile_elems += ntiles_upper(nb[m]) * TT;
            panel_elems += uint64_t(nb[m]) * TT;
            work_prefix[m + 1] = work_prefix[m] + ntiles_upper(nb[m]);
        }
        tiles.alloc(tile_elems * vbytes);
        if (with_panel) panel.alloc(panel_elems * vbytes);
        d_tile_base = upload(tile_base, s);
        d_panel_base = upload(panel_base, s);
        d_work_prefix = upload(work_prefix, s);
        d_nb = upload(nb, s);
    }
    template <class V> MatSet<V> view() const {
        MatSet<V> v;
        v.tiles = tiles.as<V>();
        v.panel = panel.as<V>();
        v.tile_base = d_tile_base.as<uint64_t>();
        v.panel_base = d_panel_base.as<uint64_t>();
        v.work_prefix = d_work_prefix.as<uint64_t>();
        v.nb = d_nb.as<uint32_t>();
        v.nmat = nmat;
        v.nb_max = nb_max;
        v.rows = world > 1 ? d_rows.as<uint32_t>() : nullptr;
        v.row_prefix = world > 1 ? d_row_prefix.as<uint64_t>() : nullptr;
        v.nrows = world > 1 ? nrows : 0;
        v.rank = rank;
        v.world = world;
        return v;
    }
    // relaxations the FW executes on the padded matrices: per k-block the
    // diagonal tile, the nb-1 panel tiles and the upper tiles off row/col kb
    uint64_t relaxations() const {
        uint64_t r = 0;
        for (uint32_t m = 0; m < nmat; ++m) r += ntiles_upper(nb[m]) * nb[m];
        return r * uint64_t(T) * T * T;
    }
    size_t bytes() const { return tiles.bytes + panel.bytes; }
};

}  // namespace

// --------------------------------------------------------------- ctx ----
struct psp_gpu_ctx {
    int device = 0;
    int rank = 0, world = 1;
    int sms = 148;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;  // world > 1 only
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
    const uint64_t n = a.tile_elems;
    const int blocks = int(std::min<uint64_t>((n + 255) / 256, uint64_t(sms) * 32));
    fill_value<V><<<std::max(blocks, 1), 256, 0, s>>>(a.tiles.as<V>(), n, Ops<V>::inf());
    CK_LAUNCH();
    if (a.nmat) {
        set_diag_zero<V><<<a.nmat, 256, 0, s>>>(a.view<V>());
        CK_LAUNCH();
    }
}

// The blocked FW driver: 3 launches per k-block on one stream.
template <class V>
void run_fw(const MatArena& a, cudaStream_t s, int sms) {
    if (a.nmat == 0 || a.nb_max == 0) return;
    set_kernel_attrs<V>();
    const MatSet<V> v = a.view<V>();
    const int smem = 2 * TT * sizeof(V);
    const uint64_t work = a.work_prefix[a.nmat];
    const int g3 = int(std::max<uint64_t>(1, std::min<uint64_t>(work, uint64_t(sms))));
    for (uint32_t kb = 0; kb < a.nb_max; ++kb) {
        fw_phase1<V><<<a.nmat, NTHREADS, 0, s>>>(v, kb);
        CK_LAUNCH();
        if (a.nb_max > 1) {
            fw_phase2<V><<<dim3(a.nmat, a.nb_max), NTHREADS, smem, s>>>(v, kb);
            CK_LAUNCH();
            fw_phase3<V><<<g3, NTHREADS, P3_SMEM<V>, s>>>(v, kb);
            CK_LAUNCH();
        }
    }
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

// Row-sharded blocked FW of the boundary graph over ctx->world GPUs
// (SURVEY §8e): tile row I is owned by rank I mod world. Per k-block the
// owner closes the diagonal tile and broadcasts it; every rank updates the
// panel tiles whose home row it owns (others contribute INF) and one
// min-allreduce assembles the full row panel; phase 3 then touches owned rows
// only. At the end every row is broadcast from its owner so each GPU holds
// the complete table (queries stay replicated, no per-query traffic).
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
    V* tiles = a.tiles.as<V>();
    // PSP_FW_PROFILE=1: per-phase CUDA-event breakdown on stderr (diagnostics)
    const bool prof = std::getenv("PSP_FW_PROFILE") != nullptr;
    const char* dm = std::getenv("PSP_DIAG_MODE");
    const bool diag_allreduce = dm && std::strcmp(dm, "allreduce") == 0;
    cudaEvent_t ev[5];
    double acc_ms[4] = {0, 0, 0, 0};
    if (prof)
        for (auto& e : ev) CK(cudaEventCreate(&e));
    for (uint32_t kb = 0; kb < nb; ++kb) {
        const int owner = int(kb % ctx->world);
        V* diag = tiles + tidx(kb, kb, nb) * TT;
        if (prof) CK(cudaEventRecord(ev[0], s));
        if (owner == ctx->rank) {
            fw_phase1<V><<<1, NTHREADS, 0, s>>>(v, kb);
            CK_LAUNCH();
        }
        if (diag_allreduce) {
            // owners contribute the closed tile, everyone else INF
            if (owner != ctx->rank) fill_value<V><<<16, 256, 0, s>>>(diag, TT, Ops<V>::inf());
            NCK(nccl().AllReduce(diag, diag, TT, dt, ncclMin, ctx->comm, s));
        } else {
            NCK(nccl().Broadcast(diag, diag, TT, dt, owner, ctx->comm, s));
        }
        if (prof) CK(cudaEventRecord(ev[1], s));
        if (nb > 1) {
            fw_phase2<V><<<dim3(1, nb), NTHREADS, smem, s>>>(v, kb);
            CK_LAUNCH();
            if (prof) CK(cudaEventRecord(ev[2], s));
            NCK(nccl().AllReduce(a.panel.p, a.panel.p, uint64_t(nb) * TT, dt, ncclMin, ctx->comm, s));
            if (prof) CK(cudaEventRecord(ev[3], s));
            if (a.nrows) {
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
                     "[psp] rank %d sharded FW nb=%u: phase1+bcast %.1f ms, phase2 %.1f ms, "
                     "allreduce %.1f ms, phase3 %.1f ms\n",
                     ctx->rank, nb, acc_ms[0], acc_ms[1], acc_ms[2], acc_ms[3]);
        for (auto& e : ev) cudaEventDestroy(e);
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

// ------------------------------------------------------------ oracle ----
struct psp_gpu_oracle {
    psp_gpu_ctx* ctx = nullptr;
    Kind kind{PSP_VALUE_U32, 0};
    double scale = 1.0;
    Reordered R;
    MatArena comps, bg;
    DBuf d_perm, d_assign, d_comp_off, d_bnd_off, d_cb_off, d_cb;
    uint64_t device_bytes = 0;
    // grow-only staging for the host-pointer query API (one call at a time;
    // the tables themselves are read-only, src/query.cpp is re-entrant too)
    std::mutex query_mu;
    DBuf query_stage;
    // grouped-query workspace (grow-only) and the event that serialises its
    // reuse across caller streams
    DBuf gw_buf, gw_bins, gw_temp, gw_tasks;
    uint64_t gw_count = 0;
    size_t gw_temp_bytes = 0;
    cudaEvent_t gw_done = nullptr;
    ~psp_gpu_oracle() {
        if (gw_done) cudaEventDestroy(gw_done);
    }
};

namespace {

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
template <class V>
void finish_query_tables(psp_gpu_oracle* o, DBuf d_bnd, cudaStream_t s) {
    const Reordered& R = o->R;
    const uint32_t k = R.k;
    std::vector<uint64_t> cb_off(k + 1, 0);
    for (uint32_t c = 0; c < k; ++c)
        cb_off[c + 1] = cb_off[c] + uint64_t(R.comp_off[c + 1] - R.comp_off[c]) *
                                        cb_stride(R.bnd_off[c + 1] - R.bnd_off[c]);
    o->d_cb.alloc(cb_off[k] * sizeof(V));
    o->d_cb_off = upload(cb_off, s);
    o->d_comp_off = upload(R.comp_off, s);
    o->d_bnd_off = std::move(d_bnd);
    o->d_perm = upload(R.perm, s);
    o->d_assign = upload(R.assign, s);
    extract_to_boundary<V><<<std::max(k, 1u), 256, 0, s>>>(
        o->comps.view<V>(), o->d_comp_off.as<uint32_t>(), o->d_bnd_off.as<uint32_t>(),
        o->d_cb_off.as<uint64_t>(), o->d_cb.as<V>());
    CK_LAUNCH();
}

template <class V>
void device_build(psp_gpu_oracle* o, psp_build_stats* st) {
    psp_gpu_ctx* ctx = o->ctx;
    cudaStream_t s = ctx->stream;
    const Reordered& R = o->R;
    const uint32_t k = R.k;
    const int q = o->kind.shift;
    EventTimer t_init, t_k1, t_k2, t_post;

    // ---- Phase 2: K0 + K1
    auto t0 = Clock::now();
    std::vector<uint64_t> sizes(k);
    for (uint32_t c = 0; c < k; ++c) sizes[c] = R.comp_off[c + 1] - R.comp_off[c];
    EdgeLists L = split_edges(R);
    t_init.start(s);
    o->comps.create(sizes, sizeof(V), true, s);
    fill_arena<V>(o->comps, s, ctx->sms);
    scatter<V>(o->comps, &L.mat, L.ii, L.jj, L.w, q, s);
    t_init.stop(s);
    t_k1.start(s);
    run_fw<V>(o->comps, s, ctx->sms);
    t_k1.stop(s);
    CK(cudaStreamSynchronize(s));
    const double k1_ms = t_k1.ms();
    double init_ms = t_init.ms();
    const double component_ms = ms_since(t0);

    // ---- Phase 3: BG init + K2 + query tables
    t0 = Clock::now();
    const uint64_t b = R.b();
    DBuf d_bnd = upload(R.bnd_off, s);
    unsigned long long clique = 0;
    double k2_ms = 0.0;
    if (b > 0) {
        t_post.start(s);
        o->bg.create({b}, sizeof(V), true, s);
        fill_arena<V>(o->bg, s, ctx->sms);
        DBuf d_clique(sizeof(unsigned long long));
        CK(cudaMemsetAsync(d_clique.p, 0, sizeof(unsigned long long), s));
        copy_boundary_blocks<V><<<k, 256, 0, s>>>(o->comps.view<V>(), d_bnd.as<uint32_t>(),
                                                  o->bg.view<V>(),
                                                  d_clique.as<unsigned long long>());
        CK_LAUNCH();
        scatter<V>(o->bg, nullptr, L.bi, L.bj, L.bw, q, s);
        CK(cudaMemcpyAsync(&clique, d_clique.p, sizeof(clique), cudaMemcpyDeviceToHost, s));
        t_post.stop(s);
        CK(cudaStreamSynchronize(s));
        init_ms += t_post.ms();
        t_k2.start(s);
        if (ctx->world > 1) run_fw_sharded<V>(o->bg, ctx);
        else run_fw<V>(o->bg, s, ctx->sms);
        t_k2.stop(s);
        CK(cudaStreamSynchronize(s));
        k2_ms = t_k2.ms();
    }
    // query-side tables
    t_post.start(s);
    finish_query_tables<V>(o, std::move(d_bnd), s);
    t_post.stop(s);
    CK(cudaStreamSynchronize(s));
    init_ms += t_post.ms();
    // panels are build-time scratch
    o->comps.panel.reset();
    o->bg.panel.reset();
    const double boundary_ms = ms_since(t0);

    o->device_bytes = o->comps.bytes() + o->bg.bytes() + o->d_cb.bytes + o->d_cb_off.bytes +
                      o->d_comp_off.bytes + o->d_bnd_off.bytes + o->d_perm.bytes +
                      o->d_assign.bytes;
    if (st) {
        st->component_apsp_ms = component_ms;
        st->boundary_ms = boundary_ms;
        st->k1_device_ms = k1_ms;
        st->k2_device_ms = k2_ms;
        st->init_device_ms = init_ms;
        st->k1_relaxations = o->comps.relaxations();
        st->k2_relaxations = b ? o->bg.relaxations() : 0;
        st->boundary_total = b;
        st->bg_edges = L.bi.size() + clique;
        uint64_t stored = 0;
        for (uint32_t c = 0; c < k; ++c)
            stored += sizes[c] * sizes[c] + (R.bnd_off[c + 1] - R.bnd_off[c]) * b;
        st->stored_entries = stored;
        st->value_kind = o->kind.kind;
        st->fixed_point_shift = o->kind.shift;
        st->device_bytes = o->device_bytes;
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
    finish_query_tables<V>(o, upload(R.bnd_off, s), s);
    CK(cudaStreamSynchronize(s));
    o->device_bytes = o->comps.bytes() + o->bg.bytes() + o->d_cb.bytes;
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

template <class V>
void launch_grouped(psp_gpu_oracle* o, const QueryView<V>& q, uint64_t count, const uint32_t* v1,
                    const uint32_t* v2, double* dist, cudaStream_t s) {
    const uint32_t nbins = o->R.k * o->R.k;
    if (!o->gw_done) CK(cudaEventCreateWithFlags(&o->gw_done, cudaEventDisableTiming));
    // the workspace is shared by all calls on this oracle: order after the
    // previous user, whatever stream it ran on
    CK(cudaStreamWaitEvent(s, o->gw_done, 0));
    if (o->gw_count < count) {
        CK(cudaStreamSynchronize(s));
        o->gw_buf.alloc(count * 7 * sizeof(uint32_t));
        o->gw_count = count;
    }
    if (o->gw_bins.bytes < size_t(nbins + 1) * 4 * sizeof(uint32_t)) {
        CK(cudaStreamSynchronize(s));
        o->gw_bins.alloc(size_t(nbins + 1) * 4 * sizeof(uint32_t));
        size_t t1 = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, t1, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                         int(nbins + 1), s));
        o->gw_temp.alloc(t1);
        o->gw_temp_bytes = t1;
    }
    GroupWork w;
    uint32_t* base = o->gw_buf.as<uint32_t>();
    w.key = base;
    w.l1 = base + o->gw_count;
    w.l2 = base + 2 * o->gw_count;
    w.best = base + 3 * o->gw_count;
    w.sorted = base + 4 * o->gw_count;
    w.s_l1 = base + 5 * o->gw_count;
    w.s_l2 = base + 6 * o->gw_count;
    uint32_t* bins = o->gw_bins.as<uint32_t>();
    w.bin_cnt = bins;
    w.bin_start = bins + (nbins + 1);
    w.task_cnt = bins + 2 * size_t(nbins + 1);
    w.task_start = bins + 3 * size_t(nbins + 1);
    w.nbins = nbins;
    CK(cudaMemsetAsync(w.bin_cnt, 0, size_t(nbins + 1) * sizeof(uint32_t), s));
    const unsigned qb = unsigned((count + 255) / 256);
    group_prep<V><<<qb, 256, 0, s>>>(q, v1, v2, count, w);
    CK_LAUNCH();
    group_tasks<<<(nbins + 1 + 255) / 256, 256, 0, s>>>(w, q.bnd_off, q.k);
    CK_LAUNCH();
    size_t tb = o->gw_temp_bytes;
    CK(cub::DeviceScan::ExclusiveSum(o->gw_temp.p, tb, w.bin_cnt, w.bin_start, int(nbins + 1), s));
    tb = o->gw_temp_bytes;
    CK(cub::DeviceScan::ExclusiveSum(o->gw_temp.p, tb, w.task_cnt, w.task_start, int(nbins + 1), s));
    // task records: upper bound on the task count without a host round trip
    {
        uint64_t max_tasks = 0;
        for (uint32_t c = 0; c < o->R.k; ++c)
            max_tasks = std::max<uint64_t>(max_tasks, (o->R.bnd_off[c + 1] - o->R.bnd_off[c] + 31) / 32);
        max_tasks *= (count + GQ - 1) / GQ + std::min<uint64_t>(count, nbins);
        if (o->gw_tasks.bytes < max_tasks * sizeof(uint4) + 16) {
            CK(cudaStreamSynchronize(s));
            o->gw_tasks.alloc(max_tasks * sizeof(uint4) + 16);
        }
    }
    w.tasks = o->gw_tasks.as<uint4>();
    group_emit<<<(nbins + 255) / 256, 256, 0, s>>>(w, q.bnd_off, q.k);
    CK_LAUNCH();
    CK(cudaMemsetAsync(w.bin_cnt, 0, size_t(nbins) * sizeof(uint32_t), s));
    group_scatter<<<qb, 256, 0, s>>>(count, w);
    CK_LAUNCH();
    const int gsmem = GWARPS * sizeof(WarpStage<V>);
    static bool attr_set[2] = {false, false};
    if (!attr_set[sizeof(V) == 4 && std::is_same<V, float>::value]) {
        CK(cudaFuncSetAttribute(query_grouped<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, gsmem));
        attr_set[std::is_same<V, float>::value] = true;
    }
    query_grouped<V><<<o->ctx->sms * 2, GTHREADS, gsmem, s>>>(q, w);
    CK_LAUNCH();
    group_finish<V><<<qb, 256, 0, s>>>(q, v1, v2, count, w, dist);
    CK_LAUNCH();
    CK(cudaEventRecord(o->gw_done, s));
}

// Every batch goes through the pair-grouped kernel: measured on cfg2/cfg3 it
// beats one-warp-per-query from 1K pairs up (8.4M vs 3.4M q/s at 1K, 393M vs
// 17M at 1M; profiles/bench/r1_kernel_crossover.jsonl). query_warp remains
// for k*k beyond 32-bit bin keys and as the PSP_QUERY_KERNEL=warp check.
constexpr double GROUP_MIN_DENSITY = 0.0;

template <class V>
void launch_queries(const psp_gpu_oracle* o, uint64_t count, const uint32_t* v1,
                    const uint32_t* v2, double* dist, cudaStream_t s, uint32_t* bad_id) {
    if (count == 0) return;
    QueryView<V> q;
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
    const uint64_t k = o->R.k;
    const double pairs = double(k) * double(k + 1) / 2.0;
    // PSP_QUERY_KERNEL=warp|grouped overrides the density heuristic (tests,
    // profiling); both kernels return identical distances.
    const char* force = std::getenv("PSP_QUERY_KERNEL");
    bool grouped = double(count) >= GROUP_MIN_DENSITY * pairs;
    if (force && std::strcmp(force, "warp") == 0) grouped = false;
    if (force && std::strcmp(force, "grouped") == 0) grouped = true;
    if (grouped && k * k < (1ull << 31) && count < (1ull << 31)) {
        launch_grouped<V>(const_cast<psp_gpu_oracle*>(o), q, count, v1, v2, dist, s);
        return;
    }
    const uint64_t warps_per_block = 8;
    const uint64_t want = (count + warps_per_block - 1) / warps_per_block;
    const unsigned blocks =
        unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(o->ctx->sms) * 16)));
    query_warp<V><<<blocks, 256, 0, s>>>(q, v1, v2, count, dist);
    CK_LAUNCH();
}

}  // namespace

// --------------------------------------------------------- PSP1 files --
struct PinnedBuf {
    void* p = nullptr;
    explicit PinnedBuf(size_t n) { CK(cudaMallocHost(&p, n)); }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

constexpr size_t IO_CHUNK = size_t(64) << 20;  // bytes per device/host staging chunk

// Append `len` bytes at device pointer d (8-byte aligned) to the running CRC:
// per-segment raw CRCs on the GPU, folded on the host.
void crc_device_bytes(Crc64Stream& crc, const uint8_t* d, uint64_t len, DBuf& seg,
                      std::vector<uint64_t>& hseg, cudaStream_t s) {
    if (len == 0) return;
    const uint64_t nseg = (len + CRC_SEG - 1) / CRC_SEG;
    if (seg.bytes < nseg * 8) seg.alloc(nseg * 8);
    crc64_segments<<<unsigned((nseg + 127) / 128), 128, 0, s>>>(d, len, crc.table(),
                                                                seg.as<uint64_t>());
    CK_LAUNCH();
    hseg.resize(nseg);
    CK(cudaMemcpyAsync(hseg.data(), seg.p, nseg * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < nseg; ++i)
        crc.append_raw(hseg[i], std::min<uint64_t>(CRC_SEG, len - i * CRC_SEG));
}

template <class V>
void save_tables(const psp_gpu_oracle* o, std::FILE* f, Crc64Stream& crc) {
    cudaStream_t s = o->ctx->stream;
    DBuf chunk(IO_CHUNK), seg;
    PinnedBuf host(IO_CHUNK);
    std::vector<uint64_t> hseg;
    auto emit = [&](const MatArena& a, uint32_t m, uint32_t row0, uint32_t nrows, uint32_t ncols) {
        if (!nrows || !ncols) return;
        const uint32_t per = uint32_t(std::max<uint64_t>(1, IO_CHUNK / (uint64_t(ncols) * 8)));
        for (uint32_t r0 = 0; r0 < nrows; r0 += per) {
            const uint32_t nr = std::min(per, nrows - r0);
            const uint64_t cnt = uint64_t(nr) * ncols, bytes = cnt * 8;
            window_to_f64<V><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(
                a.view<V>(), m, row0 + r0, nr, ncols, o->scale, chunk.as<double>());
            CK_LAUNCH();
            CK(cudaMemcpyAsync(host.p, chunk.p, bytes, cudaMemcpyDeviceToHost, s));
            crc_device_bytes(crc, chunk.as<uint8_t>(), bytes, seg, hseg, s);  // syncs
            if (std::fwrite(host.p, 1, bytes, f) != bytes) throw Fail{PSP_EIO, "oracle write failed"};
        }
    };
    const Reordered& R = o->R;
    for (uint32_t c = 0; c < R.k; ++c) {
        const uint32_t sz = R.comp_off[c + 1] - R.comp_off[c];
        emit(o->comps, c, 0, sz, sz);
    }
    for (uint32_t c = 0; c < R.k; ++c)
        emit(o->bg, 0, R.bnd_off[c], R.bnd_off[c + 1] - R.bnd_off[c], uint32_t(R.b()));
}

void put_u64s(std::vector<uint8_t>& buf, uint64_t v) {
    const size_t at = buf.size();
    buf.resize(at + 8);
    std::memcpy(buf.data() + at, &v, 8);
}

// ================================================================ C-ABI ==
extern "C" {

int psp_gpu_abi_version(void) { return PSP_GPU_ABI_VERSION; }
const char* psp_gpu_last_error(void) { return g_err.c_str(); }

int psp_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

psp_status psp_gpu_ctx_create(int device, int rank, int world, const void* nccl_id,
                              psp_gpu_ctx** out) {
    return guarded([&] {
        if (!out) throw ArgError("ctx_create: out is NULL");
        if (world < 1 || rank < 0 || rank >= world) throw ArgError("ctx_create: bad rank/world");
        if (world > 1 && !nccl_id) throw ArgError("ctx_create: world > 1 needs an NCCL id");
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw ArgError("ctx_create: no such CUDA device");
        CK(cudaSetDevice(device));
        auto c = std::make_unique<psp_gpu_ctx>();
        c->device = device;
        c->rank = rank;
        c->world = world;
        CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        if (world > 1) {
            NcclApi& api = nccl();
            if (!api.ok) throw Fail{PSP_ENCCL, api.err};
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            NCK(api.CommInitRank(&c->comm, world, id, rank));
            // NCCL connects lazily; run the collectives the sharded build
            // uses once here (every root for the 64 KB tile broadcast, a
            // panel-sized min-allreduce, the row broadcasts) so that one-time
            // setup is part of context creation, not of the first build.
            DBuf tmp(size_t(32) << 20);
            CK(cudaMemsetAsync(tmp.p, 0, tmp.bytes, c->stream));
            for (int root = 0; root < world; ++root)
                NCK(api.Broadcast(tmp.p, tmp.p, TT, ncclUint32, root, c->comm, c->stream));
            for (size_t elems : {size_t(TT), size_t(8) << 20})
                NCK(api.AllReduce(tmp.p, tmp.p, elems, ncclUint32, ncclMin, c->comm, c->stream));
            NCK(api.GroupStart());
            for (int root = 0; root < world; ++root)
                NCK(api.Broadcast(tmp.p, tmp.p, size_t(1) << 20, ncclUint32, root, c->comm, c->stream));
            NCK(api.GroupEnd());
            CK(cudaStreamSynchronize(c->stream));
        }
        *out = c.release();
    });
}

void psp_gpu_ctx_destroy(psp_gpu_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->comm) nccl().CommDestroy(ctx->comm);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

psp_status psp_gpu_nccl_unique_id(void* out128) {
    return guarded([&] {
        if (!out128) throw ArgError("nccl_unique_id: NULL output");
        NcclApi& api = nccl();
        if (!api.ok) throw Fail{PSP_ENCCL, api.err};
        static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
        ncclUniqueId id;
        NCK(api.GetUniqueId(&id));
        std::memcpy(out128, &id, sizeof(id));
    });
}

void* psp_gpu_ctx_stream(psp_gpu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

psp_status psp_gpu_build_oracle(psp_gpu_ctx* ctx, uint64_t n, uint64_t m, const uint32_t* eu,
                                const uint32_t* ev, const double* ew, uint32_t k,
                                uint32_t workers, uint64_t seed, int value_kind,
                                psp_gpu_oracle** out, psp_build_stats* stats) {
    return guarded([&] {
        if (!ctx || !out) throw ArgError("build_oracle: NULL ctx/out");
        if (workers < 1) throw ArgError("build_oracle: workers must be at least 1");
        const Csr g = build_csr(n, m, eu, ev, ew);
        auto t0 = Clock::now();
        const std::vector<uint32_t> a = partition_graph(g, k, seed, workers);
        const double part_ms = ms_since(t0);
        psp_gpu_oracle* o = build_from_csr(ctx, g, k, a, ew, m, value_kind, part_ms, stats);
        set_peak_entries(o->R, workers, stats);
        *out = o;
    });
}

psp_status psp_gpu_build_partitioned(psp_gpu_ctx* ctx, uint64_t n, uint64_t m,
                                     const uint32_t* eu, const uint32_t* ev, const double* ew,
                                     uint32_t k, const uint32_t* assignment, int value_kind,
                                     psp_gpu_oracle** out, psp_build_stats* stats) {
    return guarded([&] {
        if (!ctx || !out || (!assignment && n)) throw ArgError("build_partitioned: NULL argument");
        if (k < 1 || k > n) throw ArgError("build_partitioned: k must be in 1..n");
        const Csr g = build_csr(n, m, eu, ev, ew);
        std::vector<uint32_t> a(assignment, assignment + n);
        psp_gpu_oracle* o = build_from_csr(ctx, g, k, a, ew, m, value_kind, 0.0, stats);
        set_peak_entries(o->R, 1, stats);
        *out = o;
    });
}

psp_status psp_gpu_oracle_import(psp_gpu_ctx* ctx, uint64_t n, uint32_t k,
                                 const uint32_t* permutation, const uint32_t* assignment,
                                 const uint64_t* component_offset,
                                 const uint64_t* boundary_offset,
                                 const double* const* component_tables,
                                 const double* const* boundary_tables, int value_kind,
                                 psp_gpu_oracle** out) {
    return guarded([&] {
        if (!ctx || !out || (n && (!permutation || !assignment)) || !component_offset ||
            !boundary_offset || (k && (!component_tables || !boundary_tables)))
            throw ArgError("oracle_import: NULL argument");
        if (k < 1 || k > n) throw ArgError("oracle_import: k must be in 1..n");
        auto o = std::make_unique<psp_gpu_oracle>();
        o->ctx = ctx;
        Reordered& R = o->R;
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
        std::vector<const double*> ptr;
        std::vector<uint64_t> len;
        for (uint32_t c = 0; c < k; ++c) {
            const uint64_t s = R.comp_off[c + 1] - R.comp_off[c];
            ptr.push_back(component_tables[c]);
            len.push_back(s * s);
            ptr.push_back(boundary_tables[c]);
            len.push_back(uint64_t(R.bnd_off[c + 1] - R.bnd_off[c]) * R.b());
        }
        o->kind = choose_kind_tables(value_kind, ptr, len);
        o->scale = std::ldexp(1.0, -o->kind.shift);
        CK(cudaSetDevice(ctx->device));
        if (o->kind.kind == PSP_VALUE_U32) import_tables<uint32_t>(o.get(), component_tables, boundary_tables);
        else import_tables<float>(o.get(), component_tables, boundary_tables);
        *out = o.release();
    });
}

psp_status psp_gpu_oracle_save(const psp_gpu_oracle* o, const char* path) {
    return guarded([&] {
        if (!o || !path) throw ArgError("oracle_save: NULL argument");
        CK(cudaSetDevice(o->ctx->device));
        const Reordered& R = o->R;
        std::FILE* f = std::fopen(path, "wb");
        if (!f) throw Fail{PSP_EIO, std::string(path) + ": cannot open for writing"};
        std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
        Crc64Stream crc;
        // header and id sections (src/oracle_io.cpp:106-127)
        std::vector<uint8_t> head = {'P', 'S', 'P', '1', 1, 0, 0, 0};
        put_u64s(head, R.n);
        put_u64s(head, R.k);
        put_u64s(head, R.b());
        for (uint64_t v = 0; v < R.n; ++v) put_u64s(head, R.perm[v]);
        for (uint64_t v = 0; v < R.n; ++v) put_u64s(head, R.assign[v]);
        std::vector<uint8_t> packed((R.n + 7) / 8, 0);
        for (uint64_t v = 0; v < R.n; ++v)
            if (R.flags[v]) packed[v / 8] |= uint8_t(1u << (v % 8));
        head.insert(head.end(), packed.begin(), packed.end());
        for (uint32_t c = 0; c <= R.k; ++c) put_u64s(head, R.comp_off[c]);
        crc.update(head.data(), head.size());
        if (std::fwrite(head.data(), 1, head.size(), f) != head.size())
            throw Fail{PSP_EIO, "oracle write failed"};
        if (o->kind.kind == PSP_VALUE_U32) save_tables<uint32_t>(o, f, crc);
        else save_tables<float>(o, f, crc);
        const uint64_t sum = crc.value();
        if (std::fwrite(&sum, 1, 8, f) != 8 || std::fflush(f) != 0)
            throw Fail{PSP_EIO, "oracle write failed"};
    });
}

psp_status psp_gpu_oracle_load(psp_gpu_ctx* ctx, const char* path, int value_kind,
                               psp_gpu_oracle** out) {
    return guarded([&] {
        if (!ctx || !path || !out) throw ArgError("oracle_load: NULL argument");
        const std::string name(path);
        auto io = [&](const std::string& msg) { return Fail{PSP_EIO, name + ": " + msg}; };
        std::ifstream in(name, std::ios::binary);
        if (!in) throw io("cannot open for reading");
        in.seekg(0, std::ios::end);
        const int64_t total = in.tellg();
        in.seekg(0, std::ios::beg);
        if (total < 4 + 4 + 8) throw io("truncated oracle file");
        // validation order and messages follow read_oracle (src/oracle_io.cpp:129-255)
        uint8_t head[32] = {0};  // magic, version, n, k, b
        in.read(reinterpret_cast<char*>(head), std::min<int64_t>(32, total));
        if (std::memcmp(head, "PSP1", 4) != 0) throw Fail{PSP_EFORMAT, name + ": not an oracle file"};
        uint32_t version;
        std::memcpy(&version, head + 4, 4);
        if (version != 1)
            throw Fail{PSP_EFORMAT, name + ": unsupported oracle format version " + std::to_string(version)};
        const uint64_t payload = uint64_t(total) - 8;
        if (payload < 32) throw io("truncated oracle file");
        uint64_t n, k, b;
        std::memcpy(&n, head + 8, 8);
        std::memcpy(&k, head + 16, 8);
        std::memcpy(&b, head + 24, 8);
        const uint64_t remaining = payload - 32;
        if (n > remaining / 16 || k > remaining / 8) throw io("truncated oracle file");
        if (k < 1 || k > n || b > n || n > 0xffffffffull) throw io("inconsistent oracle header");
        const uint64_t fixed = 16 * n + (n + 7) / 8 + 8 * (k + 1);
        if (remaining < fixed) throw io("truncated oracle file");
        // read everything with the table section 8-byte aligned in memory
        const uint64_t table_at = 32 + fixed;
        const size_t pad = (8 - table_at % 8) % 8;
        std::vector<uint64_t> store((uint64_t(total) + pad + 7) / 8 + 1);
        uint8_t* buf = reinterpret_cast<uint8_t*>(store.data()) + pad;
        in.seekg(0, std::ios::beg);
        in.read(reinterpret_cast<char*>(buf), total);
        if (in.gcount() != total) throw io("truncated oracle file");
        const uint8_t* p = buf + 32;
        auto rd64 = [&](const uint8_t* q) {
            uint64_t v;
            std::memcpy(&v, q, 8);
            return v;
        };
        std::vector<uint32_t> perm(n), assign(n);
        for (uint64_t v = 0; v < n; ++v) {
            const uint64_t t = rd64(p + 8 * v);
            if (t >= n) throw io("permutation entry out of range");
            perm[v] = uint32_t(t);
        }
        p += 8 * n;
        for (uint64_t v = 0; v < n; ++v) {
            const uint64_t c = rd64(p + 8 * v);
            if (c >= k) throw io("component assignment out of range");
            assign[v] = uint32_t(c);
        }
        p += 8 * n;
        const uint8_t* packed = p;
        p += (n + 7) / 8;
        std::vector<uint64_t> co(k + 1), bo(k + 1, 0);
        for (uint64_t c = 0; c <= k; ++c) co[c] = rd64(p + 8 * c);
        p += 8 * (k + 1);
        if (co[0] != 0 || co[k] != n) throw io("inconsistent component offsets");
        for (uint64_t c = 0; c < k; ++c) {
            if (co[c + 1] < co[c] || co[c + 1] > n) throw io("inconsistent component offsets");
            bool interior = false;
            uint64_t nbnd = 0;
            for (uint64_t v = co[c]; v < co[c + 1]; ++v) {
                if (assign[v] != c) throw io("assignment does not match component offsets");
                if ((packed[v / 8] >> (v % 8)) & 1u) {
                    if (interior) throw io("boundary vertices must prefix each component");
                    ++nbnd;
                } else {
                    interior = true;
                }
            }
            bo[c + 1] = bo[c] + nbnd;
        }
        if (bo[k] != b) throw io("boundary count does not match flags");
        uint64_t table_bytes = 0;
        for (uint64_t c = 0; c < k; ++c) {
            const uint64_t sz = co[c + 1] - co[c];
            table_bytes += 8 * (sz * sz + (bo[c + 1] - bo[c]) * b);
        }
        if (payload - table_at != table_bytes)
            throw io(payload - table_at < table_bytes ? "truncated oracle file"
                                                      : "oracle file has trailing data");
        // checksum: header on the host, tables on the device
        CK(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        Crc64Stream crc;
        crc.update(buf, table_at);
        {
            DBuf chunk(IO_CHUNK), seg;
            std::vector<uint64_t> hseg;
            for (uint64_t at = 0; at < table_bytes; at += IO_CHUNK) {
                const uint64_t len = std::min<uint64_t>(IO_CHUNK, table_bytes - at);
                CK(cudaMemcpyAsync(chunk.p, buf + table_at + at, len, cudaMemcpyHostToDevice, s));
                crc_device_bytes(crc, chunk.as<uint8_t>(), len, seg, hseg, s);
            }
        }
        if (rd64(buf + payload) != crc.value())
            throw Fail{PSP_ECHECKSUM, name + ": oracle checksum mismatch"};
        std::vector<const double*> ct(k), bt(k);
        const double* tp = reinterpret_cast<const double*>(buf + table_at);
        for (uint64_t c = 0; c < k; ++c) {
            ct[c] = tp;
            tp += (co[c + 1] - co[c]) * (co[c + 1] - co[c]);
        }
        for (uint64_t c = 0; c < k; ++c) {
            bt[c] = tp;
            tp += (bo[c + 1] - bo[c]) * b;
        }
        const psp_status st = psp_gpu_oracle_import(ctx, n, uint32_t(k), perm.data(), assign.data(),
                                                    co.data(), bo.data(), ct.data(), bt.data(),
                                                    value_kind, out);
        if (st != PSP_OK) throw Fail{st, g_err};
    });
}

void psp_gpu_oracle_free(psp_gpu_oracle* o) {
    if (!o) return;
    cudaSetDevice(o->ctx->device);
    delete o;
}

psp_status psp_gpu_oracle_info(const psp_gpu_oracle* o, psp_oracle_info* out) {
    return guarded([&] {
        if (!o || !out) throw ArgError("oracle_info: NULL argument");
        out->n = o->R.n;
        out->k = o->R.k;
        out->b = o->R.b();
        out->value_kind = o->kind.kind;
        out->fixed_point_shift = o->kind.shift;
        out->device = o->ctx->device;
        out->tile = T;
    });
}

psp_status psp_gpu_oracle_ids(const psp_gpu_oracle* o, uint32_t* permutation,
                              uint32_t* inverse_permutation, uint32_t* assignment,
                              uint8_t* boundary_flags, uint64_t* component_offset,
                              uint64_t* boundary_offset, uint32_t* boundary_vertex) {
    return guarded([&] {
        if (!o) throw ArgError("oracle_ids: NULL oracle");
        const Reordered& R = o->R;
        if (permutation) std::copy(R.perm.begin(), R.perm.end(), permutation);
        if (inverse_permutation) std::copy(R.inv.begin(), R.inv.end(), inverse_permutation);
        if (assignment) std::copy(R.assign.begin(), R.assign.end(), assignment);
        if (boundary_flags) std::copy(R.flags.begin(), R.flags.end(), boundary_flags);
        if (component_offset) std::copy(R.comp_off.begin(), R.comp_off.end(), component_offset);
        if (boundary_offset) std::copy(R.bnd_off.begin(), R.bnd_off.end(), boundary_offset);
        if (boundary_vertex) {
            // boundary id -> reordered vertex (src/oracle.cpp:80-85)
            uint64_t at = 0;
            for (uint64_t v = 0; v < R.n; ++v)
                if (R.flags[v]) boundary_vertex[at++] = static_cast<uint32_t>(v);
        }
    });
}

psp_status psp_gpu_export_component(const psp_gpu_oracle* o, uint32_t c, double* dst) {
    return guarded([&] {
        if (!o || !dst) throw ArgError("export_component: NULL argument");
        if (c >= o->R.k) throw ArgError("export_component: component out of range");
        const uint32_t s = o->R.comp_off[c + 1] - o->R.comp_off[c];
        if (o->kind.kind == PSP_VALUE_U32) export_window<uint32_t>(o, o->comps, c, 0, s, s, dst);
        else export_window<float>(o, o->comps, c, 0, s, s, dst);
    });
}

psp_status psp_gpu_export_boundary_rows(const psp_gpu_oracle* o, uint32_t c, double* dst) {
    return guarded([&] {
        if (!o || !dst) throw ArgError("export_boundary_rows: NULL argument");
        if (c >= o->R.k) throw ArgError("export_boundary_rows: component out of range");
        const uint32_t g = o->R.bnd_off[c], B = o->R.bnd_off[c + 1] - g;
        const uint32_t b = static_cast<uint32_t>(o->R.b());
        if (B == 0 || b == 0) return;
        if (o->kind.kind == PSP_VALUE_U32) export_window<uint32_t>(o, o->bg, 0, g, B, b, dst);
        else export_window<float>(o, o->bg, 0, g, B, b, dst);
    });
}

psp_status psp_gpu_query_batch(const psp_gpu_oracle* o, uint64_t count, const uint32_t* v1,
                               const uint32_t* v2, double* dist, uint64_t* minplus_ops) {
    return guarded([&] {
        if (!o) throw ArgError("query_batch: NULL oracle");
        if (count == 0) return;
        if (!v1 || !v2 || !dist) throw ArgError("query_batch: NULL array");
        const Reordered& R = o->R;
        cudaStream_t s = o->ctx->stream;
        CK(cudaSetDevice(o->ctx->device));
        psp_gpu_oracle* mo = const_cast<psp_gpu_oracle*>(o);
        std::lock_guard<std::mutex> lock(mo->query_mu);
        // ids are range-checked on the device (src/query.cpp:30 semantics:
        // any bad id -> PSP_EINVAL and no output)
        const size_t need = count * (sizeof(double) + 2 * sizeof(uint32_t)) + 16;
        if (mo->query_stage.bytes < need) mo->query_stage.alloc(need);
        double* dd = mo->query_stage.as<double>();
        uint32_t* d1 = reinterpret_cast<uint32_t*>(dd + count);
        uint32_t* d2 = d1 + count;
        uint32_t* dbad = d2 + count;
        CK(cudaMemsetAsync(dbad, 0, sizeof(uint32_t), s));
        CK(cudaMemcpyAsync(d1, v1, count * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d2, v2, count * 4, cudaMemcpyHostToDevice, s));
        if (o->kind.kind == PSP_VALUE_U32) launch_queries<uint32_t>(o, count, d1, d2, dd, s, dbad);
        else launch_queries<float>(o, count, d1, d2, dd, s, dbad);
        uint32_t bad = 0;
        CK(cudaMemcpyAsync(&bad, dbad, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (bad) throw ArgError("query: vertex id out of range");  // src/query.cpp:30
        CK(cudaMemcpyAsync(dist, dd, count * 8, cudaMemcpyDeviceToHost, s));
        if (minplus_ops) {
            for (uint64_t i = 0; i < count; ++i) {
                const uint32_t c1 = R.assign[R.perm[v1[i]]], c2 = R.assign[R.perm[v2[i]]];
                const uint64_t b1 = R.bnd_off[c1 + 1] - R.bnd_off[c1];
                const uint64_t b2 = R.bnd_off[c2 + 1] - R.bnd_off[c2];
                minplus_ops[i] = b1 * b2 + b2;  // src/query.cpp:73
            }
        }
        CK(cudaStreamSynchronize(s));
    });
}

psp_status psp_gpu_query_batch_device(const psp_gpu_oracle* o, uint64_t count,
                                      const uint32_t* v1, const uint32_t* v2, double* dist,
                                      void* stream) {
    return guarded([&] {
        if (!o) throw ArgError("query_batch_device: NULL oracle");
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : o->ctx->stream;
        if (o->kind.kind == PSP_VALUE_U32) launch_queries<uint32_t>(o, count, v1, v2, dist, s, nullptr);
        else launch_queries<float>(o, count, v1, v2, dist, s, nullptr);
    });
}

psp_status psp_gpu_apsp_dense(psp_gpu_ctx* ctx, uint64_t n, uint64_t m, const uint32_t* eu,
                              const uint32_t* ev, const double* ew, uint64_t block_size,
                              int value_kind, double* out) {
    return guarded([&] {
        if (!ctx) throw ArgError("apsp_dense: NULL ctx");
        const Csr g = build_csr(n, m, eu, ev, ew);
        if (n == 0) return;
        if (block_size == 0) throw ArgError("apsp_dense: block size must be positive");
        const Kind kind = choose_kind(value_kind, ew, m, n);
        CK(cudaSetDevice(ctx->device));
        if (kind.kind == PSP_VALUE_U32) dense_apsp<uint32_t>(ctx, g, ew, m, kind, out);
        else dense_apsp<float>(ctx, g, ew, m, kind, out);
    });
}

psp_status psp_gpu_boundary_apsp(psp_gpu_ctx* ctx, uint64_t b, uint64_t m, const uint32_t* eu,
                                 const uint32_t* ev, const double* ew, int value_kind,
                                 double* out) {
    // The boundary graph's all-pairs table is exactly the dense APSP of the
    // boundary graph; rows are already in boundary-id (component) order.
    return psp_gpu_apsp_dense(ctx, b, m, eu, ev, ew, 64, value_kind, out);
}

psp_status psp_gpu_minplus_peak(psp_gpu_ctx* ctx, int value_kind, double* relax_per_s,
                                double* sm_clock_mhz) {
    return guarded([&] {
        if (!ctx || !relax_per_s) throw ArgError("minplus_peak: NULL argument");
        CK(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        DBuf out(ctx->sms * 64 * sizeof(uint32_t));
        const int blocks = ctx->sms * 4;
        const uint32_t iters = 1 << 14;
        EventTimer t;
        for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
            t.start(s);
            if (value_kind == PSP_VALUE_F32)
                minplus_peak_kernel<float><<<blocks, NTHREADS, 0, s>>>(out.as<float>(), iters, 1.0f);
            else
                minplus_peak_kernel<uint32_t><<<blocks, NTHREADS, 0, s>>>(out.as<uint32_t>(), iters, 1u);
            CK_LAUNCH();
            t.stop(s);
        }
        const double ms = t.ms();
        *relax_per_s = double(blocks) * NTHREADS * 64.0 * iters / (ms * 1e-3);
        if (sm_clock_mhz) {
            int khz = 0;
            CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, ctx->device));
            *sm_clock_mhz = khz / 1000.0;
        }
    });
}

psp_status psp_partition_graph(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                               const double* ew, uint32_t k, uint64_t seed, uint32_t threads,
                               uint32_t* assignment) {
    return guarded([&] {
        const Csr g = build_csr(n, m, eu, ev, ew);
        const std::vector<uint32_t> a = partition_graph(g, k, seed, std::max(1u, threads));
        std::copy(a.begin(), a.end(), assignment);
    });
}

psp_status psp_generate_grid(int kind, uint64_t rows, uint64_t cols, int unit, double lo,
                             double hi, uint64_t seed, uint64_t* m, uint32_t* eu, uint32_t* ev,
                             double* ew) {
    return guarded([&] {
        if (!m) throw ArgError("generate_grid: NULL m");
        if (kind != 0 && kind != 1) throw ArgError("generate_grid: kind must be 0 or 1");
        if (!eu) {
            if (rows == 0 || cols == 0) throw ArgError("grid dimensions must be positive");
            *m = rows * (cols - 1) + (rows - 1) * cols + (kind == 1 ? (rows - 1) * (cols - 1) : 0);
            return;
        }
        std::vector<uint32_t> a, b;
        std::vector<double> w;
        generate_grid(kind, rows, cols, unit != 0, lo, hi, seed, a, b, w);
        std::copy(a.begin(), a.end(), eu);
        std::copy(b.begin(), b.end(), ev);
        std::copy(w.begin(), w.end(), ew);
        *m = a.size();
    });
}

void psp_random_pairs(uint64_t n, uint64_t count, uint64_t seed, uint32_t* v1, uint32_t* v2) {
    std::mt19937_64 rng(seed);
    for (uint64_t i = 0; i < count; ++i) {
        v1[i] = static_cast<uint32_t>(rng() % n);
        v2[i] = static_cast<uint32_t>(rng() % n);
    }
}

}  // extern "C"

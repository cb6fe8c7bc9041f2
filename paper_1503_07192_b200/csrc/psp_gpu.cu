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
//
// Layout of the library (one translation unit):
//   minplus.cuh, fw_kernels.cuh, query_kernels.cuh, oracle_file.cuh  kernels
//   engine_runtime.cuh   error plumbing, device buffers, tile arenas
//   engine_fw.cuh        contexts, FW drivers (1 GPU / row-sharded NCCL)
//   engine_oracle.cuh    device oracle: build, import, export, query launch
//   engine_file.cuh      PSP1 files from/to device tables
//   engine_shard.cuh     routed (sharded) queries over NVLink
//   engine_graphio.cuh   graph text parsed on the GPU (load_graph), writer
//   psp_gpu.cu           this file: the extern "C" entry points
//   host_graph.cpp, partition.cpp   host graph plumbing and partitioner
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <future>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <random>
#include <thread>
#include <type_traits>
#include <string>
#include <vector>

#include "bg_order.hpp"
#include "fw_kernels.cuh"
#include "host_graph.hpp"
#include "k1_order.hpp"
#include "minplus.cuh"
#include "nccl_api.hpp"
#include "oracle_file.cuh"
#include "psp_gpu.h"
#include "query_kernels.cuh"

using namespace pspg;

#include "engine_runtime.cuh"
#include "engine_fw.cuh"
#include "engine_oracle.cuh"
#include "engine_file.cuh"
#include "engine_shard.cuh"
#include "engine_graphio.cuh"

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
    buf_cache().flush();
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

psp_status psp_gpu_alloc_stats(uint64_t* out4) {
    return guarded([&] {
        if (!out4) throw ArgError("alloc_stats: NULL output");
        out4[0] = g_malloc_ns.load();
        out4[1] = g_malloc_calls.load();
        out4[2] = g_free_ns.load();
        out4[3] = g_free_calls.load();
    });
}

psp_status psp_gpu_ctx_set_boundary_storage(psp_gpu_ctx* ctx, int storage) {
    return guarded([&] {
        if (!ctx) throw ArgError("ctx_set_boundary_storage: NULL ctx");
        if (storage != PSP_STORAGE_REPLICATED && storage != PSP_STORAGE_ROW_SHARDED)
            throw ArgError("ctx_set_boundary_storage: storage must be PSP_STORAGE_REPLICATED or "
                           "PSP_STORAGE_ROW_SHARDED");
        if (storage == PSP_STORAGE_ROW_SHARDED && !vmm_api().ok)
            throw Fail{PSP_ECUDA, "ctx_set_boundary_storage: CUDA virtual memory management unavailable"};
        ctx->storage = storage;
    });
}

psp_status psp_gpu_build_oracle(psp_gpu_ctx* ctx, uint64_t n, uint64_t m, const uint32_t* eu,
                                const uint32_t* ev, const double* ew, uint32_t k,
                                uint32_t workers, uint64_t seed, int value_kind,
                                psp_gpu_oracle** out, psp_build_stats* stats) {
    return guarded([&] {
        if (!ctx || !out) throw ArgError("build_oracle: NULL ctx/out");
        if (workers < 1) throw ArgError("build_oracle: workers must be at least 1");
        const Csr g = build_csr(n, m, eu, ev, ew);
        auto t0 = Clock::now();
        // multi-GPU: the partition is deterministic (workers never change it,
        // include/psp/oracle.hpp:80-84), so rank 0 computes it with all host
        // threads and broadcasts it instead of every rank competing for the
        // same cores
        std::vector<uint32_t> a;
        if (ctx->world > 1) {
            CK(cudaSetDevice(ctx->device));
            uint64_t ok = 1;
            std::exception_ptr err;  // rank 0's failure, rethrown after the broadcast
            if (ctx->rank == 0) {
                try {
                    a = partition_graph(g, k, seed, workers);
                } catch (...) {
                    ok = 0;
                    err = std::current_exception();
                }
            }
            DBuf d((size_t(n) + 2) * 4);
            if (ctx->rank == 0) {
                if (ok) CK(cudaMemcpyAsync(d.as<uint32_t>() + 2, a.data(), size_t(n) * 4, cudaMemcpyHostToDevice, ctx->stream));
                CK(cudaMemcpyAsync(d.p, &ok, 8, cudaMemcpyHostToDevice, ctx->stream));
            }
            NCK(nccl().Broadcast(d.p, d.p, (size_t(n) + 2) * 4, ncclUint8, 0, ctx->comm, ctx->stream));
            CK(cudaMemcpyAsync(&ok, d.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            if (err) std::rethrow_exception(err);
            if (!ok) throw ArgError("partition_graph failed on rank 0");
            a.resize(n);
            CK(cudaMemcpyAsync(a.data(), d.as<uint32_t>() + 2, size_t(n) * 4, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        } else {
            a = partition_graph(g, k, seed, workers);
        }
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
        reordered_from_ids(R, n, k, permutation, assignment, component_offset, boundary_offset);
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
        require_replicated(o, "oracle_save");
        CK(cudaSetDevice(o->ctx->device));
        const Reordered& R = o->R;
        const int fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (fd < 0) throw Fail{PSP_EIO, std::string(path) + ": cannot open for writing"};
        struct Fd {
            int fd;
            ~Fd() { ::close(fd); }
        } fd_guard{fd};
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
        pwrite_all(fd, head.data(), head.size(), 0);
        const uint64_t end = o->kind.kind == PSP_VALUE_U32 ? save_tables<uint32_t>(o, fd, head.size(), crc)
                                                          : save_tables<float>(o, fd, head.size(), crc);
        const uint64_t sum = crc.value();
        pwrite_all(fd, &sum, 8, end);
    });
}

psp_status psp_gpu_oracle_load(psp_gpu_ctx* ctx, const char* path, int value_kind,
                               psp_gpu_oracle** out) {
    return guarded([&] {
        if (!ctx || !path || !out) throw ArgError("oracle_load: NULL argument");
        if (value_kind != PSP_VALUE_AUTO && value_kind != PSP_VALUE_U32 && value_kind != PSP_VALUE_F32)
            throw ArgError("value_kind must be PSP_VALUE_AUTO, PSP_VALUE_U32 or PSP_VALUE_F32");
        const std::string name(path);
        auto io = [&](const std::string& msg) { return Fail{PSP_EIO, name + ": " + msg}; };
        const int fd = ::open(path, O_RDONLY);
        if (fd < 0) throw io("cannot open for reading");
        struct Fd {
            int fd;
            ~Fd() { ::close(fd); }
        } fd_guard{fd};
        struct stat sb {};
        if (::fstat(fd, &sb) != 0) throw io("cannot open for reading");
        const int64_t total = sb.st_size;
        if (total < 4 + 4 + 8) throw io("truncated oracle file");
        // validation order and messages follow read_oracle (src/oracle_io.cpp:129-255)
        uint8_t head[32] = {0};  // magic, version, n, k, b
        pread_all(fd, head, uint64_t(std::min<int64_t>(32, total)), 0, name);
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
        // the header and id sections on the host; the tables stream to the device
        const uint64_t table_at = 32 + fixed;
        std::vector<uint8_t> hdr(table_at);
        pread_all(fd, hdr.data(), table_at, 0, name);
        const uint8_t* p = hdr.data() + 32;
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
        CK(cudaSetDevice(ctx->device));
        auto o = std::make_unique<psp_gpu_oracle>();
        o->ctx = ctx;
        reordered_from_ids(o->R, n, uint32_t(k), perm.data(), assign.data(), co.data(), bo.data());
        cudaStream_t s = ctx->stream;
        std::vector<uint64_t> sizes(k);
        for (uint64_t c = 0; c < k; ++c) sizes[c] = co[c + 1] - co[c];
        // one streamed pass: CRC + conversion (u32 at q = 0 unless f32 is
        // asked for) + the kind analysis; a second pass converts again only
        // when the tables need another kind (fractional or huge weights)
        auto pass = [&](bool f32, int shift, Crc64Stream* crc) {
            const size_t vb = 4;
            o->comps.create(sizes, vb, false, s);
            if (b > 0) o->bg.create({b}, vb, false, s);
            else o->bg = MatArena();
            if (f32) {
                fill_arena<float>(o->comps, s, ctx->sms);
                if (b > 0) fill_arena<float>(o->bg, s, ctx->sms);
                return stream_psp1_tables<float>(o.get(), fd, name, table_at, table_bytes, shift, crc);
            }
            fill_arena<uint32_t>(o->comps, s, ctx->sms);
            if (b > 0) fill_arena<uint32_t>(o->bg, s, ctx->sms);
            return stream_psp1_tables<uint32_t>(o.get(), fd, name, table_at, table_bytes, shift, crc);
        };
        Crc64Stream crc;
        crc.update(hdr.data(), table_at);
        const Psp1Analysis a = pass(value_kind == PSP_VALUE_F32, 0, &crc);
        uint64_t stored = 0;
        pread_all(fd, &stored, 8, payload, name);
        if (stored != crc.value()) throw Fail{PSP_ECHECKSUM, name + ": oracle checksum mismatch"};
        // choose_kind_tables: the smallest q with every finite entry integral
        // at 2^q, if 2 * max * 2^q stays below INF
        Kind kind{PSP_VALUE_F32, 0};
        if (value_kind != PSP_VALUE_F32) {
            const int q = a.need_q;
            if (q <= 24 && 2.0 * a.maxv * std::ldexp(1.0, q) < double(U32_INF)) kind = {PSP_VALUE_U32, q};
            else if (value_kind == PSP_VALUE_U32)
                throw Fail{PSP_EOVERFLOW, "import: tables are not exact in u32 fixed point"};
            if (kind.kind != PSP_VALUE_U32 || kind.shift != 0)
                pass(kind.kind == PSP_VALUE_F32, kind.shift, nullptr);
        }
        o->kind = kind;
        o->scale = std::ldexp(1.0, -kind.shift);
        if (kind.kind == PSP_VALUE_U32) finish_import<uint32_t>(o.get());
        else finish_import<float>(o.get());
        *out = o.release();
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
        require_replicated(o, "export_boundary_rows");
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
        require_replicated(o, "query_batch");
        if (count == 0) return;
        if (!v1 || !v2 || !dist) throw ArgError("query_batch: NULL array");
        const Reordered& R = o->R;
        cudaStream_t s = o->ctx->stream;
        CK(cudaSetDevice(o->ctx->device));
        psp_gpu_oracle* mo = const_cast<psp_gpu_oracle*>(o);
        std::lock_guard<std::mutex> lock(mo->query_mu);
        // a handful of pairs: the resident point-query server (no launch,
        // no stream sync); ids are range-checked on the device
        // (src/query.cpp:30 semantics: any bad id -> PSP_EINVAL)
        if (count <= uint64_t(MAILBOX_PAIRS)) {
            const bool served = o->kind.kind == PSP_VALUE_U32
                                    ? point_queries<uint32_t>(mo, count, v1, v2, dist)
                                    : point_queries<float>(mo, count, v1, v2, dist);
            if (served) {
                if (minplus_ops) {
                    for (uint64_t i = 0; i < count; ++i) {
                        const uint32_t c1 = R.assign[R.perm[v1[i]]], c2 = R.assign[R.perm[v2[i]]];
                        const uint64_t b1 = R.bnd_off[c1 + 1] - R.bnd_off[c1];
                        const uint64_t b2 = R.bnd_off[c2 + 1] - R.bnd_off[c2];
                        minplus_ops[i] = b1 * b2 + b2;  // src/query.cpp:73
                    }
                }
                return;
            }
        }
        auto ops = [&] {
            if (!minplus_ops) return;
            for (uint64_t i = 0; i < count; ++i) {
                const uint32_t c1 = R.assign[R.perm[v1[i]]], c2 = R.assign[R.perm[v2[i]]];
                const uint64_t b1 = R.bnd_off[c1 + 1] - R.bnd_off[c1];
                const uint64_t b2 = R.bnd_off[c2 + 1] - R.bnd_off[c2];
                minplus_ops[i] = b1 * b2 + b2;  // src/query.cpp:73
            }
        };
        const size_t need = count * (sizeof(double) + 2 * sizeof(uint32_t)) + 16;
        if (mo->query_stage.bytes < need) mo->query_stage.alloc(need);
        double* dd = mo->query_stage.as<double>();
        uint32_t* d1 = reinterpret_cast<uint32_t*>(dd + count);
        uint32_t* d2 = d1 + count;
        uint32_t* dbad = d2 + count;
        if (count <= psp_gpu_oracle::kPinnedPairs) {
            // device staging is [dist | v1 | v2 | bad]: the pairs go in with one
            // copy from pinned memory, [dist | ... | bad] come back in two, one sync
            if (mo->host_stage_bytes < need) {
                if (mo->host_stage) cudaFreeHost(mo->host_stage);
                mo->host_stage = nullptr;
                mo->host_stage_bytes = 0;
                CK(cudaMallocHost(&mo->host_stage, need));
                mo->host_stage_bytes = need;
            }
            double* hd = static_cast<double*>(mo->host_stage);
            uint32_t* h1 = reinterpret_cast<uint32_t*>(hd + count);
            std::memcpy(h1, v1, count * 4);
            std::memcpy(h1 + count, v2, count * 4);
            h1[2 * count] = 0;  // bad flag
            CK(cudaMemcpyAsync(d1, h1, (2 * count + 1) * 4, cudaMemcpyHostToDevice, s));
            if (o->kind.kind == PSP_VALUE_U32) launch_queries<uint32_t>(o, count, d1, d2, dd, s, dbad);
            else launch_queries<float>(o, count, d1, d2, dd, s, dbad);
            CK(cudaMemcpyAsync(hd, dd, count * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(h1 + 2 * count, dbad, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (h1[2 * count]) throw ArgError("query: vertex id out of range");  // src/query.cpp:30
            std::memcpy(dist, hd, count * 8);
            ops();
            return;
        }
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
        ops();
        CK(cudaStreamSynchronize(s));
    });
}

// ------------------------------------------------ pipelined host batches --
struct psp_gpu_query_pipe {
    const psp_gpu_oracle* o = nullptr;
    cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
    struct Slot {
        DBuf buf;  // dist (f64) | v1 | v2 | bad flag
        cudaEvent_t in_done{}, cmp_done{}, out_done{};
        uint32_t* h_bad = nullptr;  // pinned: the batch's bad-id flag
        bool busy = false;
    };
    std::vector<Slot> slots;
    uint64_t next = 0;
    bool bad = false;
    ~psp_gpu_query_pipe() {
        for (auto& sl : slots) {
            if (sl.busy) cudaEventSynchronize(sl.out_done);
            cudaEventDestroy(sl.in_done);
            cudaEventDestroy(sl.cmp_done);
            cudaEventDestroy(sl.out_done);
            if (sl.h_bad) cudaFreeHost(sl.h_bad);
        }
        for (cudaStream_t s : {s_in, s_cmp, s_out})
            if (s) cudaStreamDestroy(s);
    }
    void retire(Slot& sl) {
        if (!sl.busy) return;
        CK(cudaEventSynchronize(sl.out_done));
        if (*sl.h_bad) bad = true;
        sl.busy = false;
    }
};

psp_status psp_gpu_query_pipe_create(const psp_gpu_oracle* o, int depth, psp_gpu_query_pipe** out) {
    return guarded([&] {
        if (!o || !out) throw ArgError("query_pipe_create: NULL argument");
        if (depth < 1 || depth > 64) throw ArgError("query_pipe_create: depth must be in 1..64");
        require_replicated(o, "query_pipe_create");
        CK(cudaSetDevice(o->ctx->device));
        auto p = std::make_unique<psp_gpu_query_pipe>();
        p->o = o;
        for (cudaStream_t* s : {&p->s_in, &p->s_cmp, &p->s_out})
            CK(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
        p->slots.resize(depth);
        for (auto& sl : p->slots) {
            CK(cudaEventCreateWithFlags(&sl.in_done, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&sl.cmp_done, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&sl.out_done, cudaEventDisableTiming));
            CK(cudaMallocHost(&sl.h_bad, sizeof(uint32_t)));
            *sl.h_bad = 0;
        }
        *out = p.release();
    });
}

psp_status psp_gpu_query_pipe_submit(psp_gpu_query_pipe* p, uint64_t count, const uint32_t* v1,
                                     const uint32_t* v2, double* dist) {
    return guarded([&] {
        if (!p) throw ArgError("query_pipe_submit: NULL pipe");
        if (count == 0) return;
        if (!v1 || !v2 || !dist) throw ArgError("query_pipe_submit: NULL array");
        const psp_gpu_oracle* o = p->o;
        CK(cudaSetDevice(o->ctx->device));
        auto& sl = p->slots[p->next++ % p->slots.size()];
        p->retire(sl);  // its previous batch (buffers are reused)
        const size_t need = count * (sizeof(double) + 2 * sizeof(uint32_t)) + 16;
        if (sl.buf.bytes < need) sl.buf.alloc(need);
        double* dd = sl.buf.as<double>();
        uint32_t* d1 = reinterpret_cast<uint32_t*>(dd + count);
        uint32_t* d2 = d1 + count;
        uint32_t* dbad = d2 + count;
        CK(cudaMemsetAsync(dbad, 0, sizeof(uint32_t), p->s_in));
        CK(cudaMemcpyAsync(d1, v1, count * 4, cudaMemcpyHostToDevice, p->s_in));
        CK(cudaMemcpyAsync(d2, v2, count * 4, cudaMemcpyHostToDevice, p->s_in));
        CK(cudaEventRecord(sl.in_done, p->s_in));
        CK(cudaStreamWaitEvent(p->s_cmp, sl.in_done, 0));
        {
            // the oracle's group workspace is shared with the other query
            // entry points (its host-side growth is guarded here)
            psp_gpu_oracle* mo = const_cast<psp_gpu_oracle*>(o);
            std::lock_guard<std::mutex> lock(mo->query_mu);
            if (o->kind.kind == PSP_VALUE_U32) launch_queries<uint32_t>(o, count, d1, d2, dd, p->s_cmp, dbad);
            else launch_queries<float>(o, count, d1, d2, dd, p->s_cmp, dbad);
        }
        CK(cudaEventRecord(sl.cmp_done, p->s_cmp));
        CK(cudaStreamWaitEvent(p->s_out, sl.cmp_done, 0));
        CK(cudaMemcpyAsync(dist, dd, count * 8, cudaMemcpyDeviceToHost, p->s_out));
        CK(cudaMemcpyAsync(sl.h_bad, dbad, sizeof(uint32_t), cudaMemcpyDeviceToHost, p->s_out));
        CK(cudaEventRecord(sl.out_done, p->s_out));
        sl.busy = true;
    });
}

psp_status psp_gpu_query_pipe_wait(psp_gpu_query_pipe* p) {
    return guarded([&] {
        if (!p) throw ArgError("query_pipe_wait: NULL pipe");
        CK(cudaSetDevice(p->o->ctx->device));
        for (auto& sl : p->slots) p->retire(sl);
        const bool bad = p->bad;
        p->bad = false;
        if (bad) throw ArgError("query: vertex id out of range");  // src/query.cpp:30
    });
}

void psp_gpu_query_pipe_destroy(psp_gpu_query_pipe* p) {
    if (!p) return;
    cudaSetDevice(p->o->ctx->device);  // the slots' buffers belong to the oracle's device
    delete p;
}

psp_status psp_gpu_query_batch_device(const psp_gpu_oracle* o, uint64_t count,
                                      const uint32_t* v1, const uint32_t* v2, double* dist,
                                      void* stream) {
    return guarded([&] {
        if (!o) throw ArgError("query_batch_device: NULL oracle");
        require_replicated(o, "query_batch_device");
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : o->ctx->stream;
        CK(cudaSetDevice(o->ctx->device));
        // concurrent callers: the enqueue (workspace lookup and growth) is
        // serialised; their batches then run on their own streams with
        // their own workspaces
        psp_gpu_oracle* mo = const_cast<psp_gpu_oracle*>(o);
        std::lock_guard<std::mutex> lock(mo->query_mu);
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

// ------------------------------------------------------ routed queries --
psp_status psp_place_components(uint32_t k, uint32_t p, int policy, uint32_t* owner) {
    return guarded([&] {
        if (!owner) throw ArgError("place_components: NULL owner");
        const std::vector<uint32_t> o = place(k, p, policy);
        std::copy(o.begin(), o.end(), owner);
    });
}

psp_status psp_gpu_shard_create(const psp_gpu_oracle* o, const uint32_t* owner,
                                psp_gpu_shard** out) {
    return guarded([&] {
        if (!o || !owner || !out) throw ArgError("shard_create: NULL argument");
        *out = nullptr;
        psp_gpu_ctx* ctx = o->ctx;
        if (ctx->world > 1 && !ctx->comm) throw ArgError("shard_create: context has no communicator");
        CK(cudaSetDevice(ctx->device));
        auto sh = std::make_unique<psp_gpu_shard>();
        sh->ctx = ctx;
        sh->kind = o->kind;
        sh->scale = o->scale;
        sh->n = o->R.n;
        sh->k = o->R.k;
        sh->b = o->R.b();
        sh->bnd_off = o->R.bnd_off;
        sh->owner.assign(owner, owner + o->R.k);
        for (uint32_t w : sh->owner)
            if (w >= uint32_t(ctx->world)) throw ArgError("shard_create: owner >= world size");
        if (o->R.k * uint64_t(o->R.k) >= (1ull << 31))
            throw ArgError("shard_create: k * k must fit the grouped kernel's 31-bit pair keys");
        if (o->kind.kind == PSP_VALUE_U32) shard_build<uint32_t>(sh.get(), o);
        else shard_build<float>(sh.get(), o);
        *out = sh.release();
    });
}

psp_status psp_gpu_shard_free(psp_gpu_shard* sh) {
    return guarded([&] {
        if (!sh) return;
        std::unique_ptr<psp_gpu_shard> own(sh);
        psp_gpu_ctx* ctx = sh->ctx;
        CK(cudaSetDevice(ctx->device));
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->world > 1) {  // nobody may still be reading our arena
            DBuf one(4);
            CK(cudaMemsetAsync(one.p, 0, 4, ctx->stream));
            nccl_check(pspg::nccl().AllReduce(one.p, one.p, 1, ncclUint32, ncclMax, ctx->comm,
                                              ctx->stream),
                       "ncclAllReduce(shard barrier)");
            CK(cudaStreamSynchronize(ctx->stream));
        }
    });
}

psp_status psp_gpu_shard_bytes(const psp_gpu_shard* sh, uint64_t* bytes) {
    return guarded([&] {
        if (!sh || !bytes) throw ArgError("shard_bytes: NULL argument");
        *bytes = sh->device_bytes;
    });
}

psp_status psp_gpu_routed_query_batch(psp_gpu_shard* sh, uint64_t count, const uint32_t* v1,
                                      const uint32_t* v2, double* dist, uint32_t* executed_on,
                                      uint32_t* column_owner, uint32_t* transfer_entries,
                                      psp_routed_stats* stats) {
    return guarded([&] {
        if (!sh) throw ArgError("routed_query_batch: NULL shard");
        if (count && (!v1 || !v2 || !dist)) throw ArgError("routed_query_batch: NULL array");
        if (count >= (1ull << 31)) throw ArgError("routed_query_batch: count must be < 2^31");
        CK(cudaSetDevice(sh->ctx->device));
        std::lock_guard<std::mutex> lock(sh->mu);
        if (sh->kind.kind == PSP_VALUE_U32)
            routed_batch<uint32_t>(sh, count, v1, v2, dist, executed_on, column_owner,
                                   transfer_entries, stats);
        else
            routed_batch<float>(sh, count, v1, v2, dist, executed_on, column_owner,
                                transfer_entries, stats);
    });
}

// ----------------------------------------------------- graph ingestion --
namespace {
psp_graph* finish_graph(ParsedGraph&& G) {
    auto g = std::make_unique<psp_graph>();
    g->n = G.n;
    g->eu = std::move(G.eu);
    g->ev = std::move(G.ev);
    g->ew = std::move(G.ew);
    return g.release();
}

uint64_t count_lines(const DevText& t) {
    // getline's line count (the wrapped Graph error's line number)
    uint64_t nl = 0;
    for (uint64_t i = 0; i < t.len; ++i) nl += t.host[i] == '\n';
    const uint64_t lines = nl + (t.len && t.host[t.len - 1] != '\n' ? 1 : 0);
    return lines ? lines : 1;
}

psp_graph* parse_text(psp_gpu_ctx* ctx, const DevText& t, int format, const std::string& name) {
    if (format != PSP_FORMAT_EDGE_LIST && format != PSP_FORMAT_DIMACS)
        throw ArgError("graph format must be PSP_FORMAT_EDGE_LIST or PSP_FORMAT_DIMACS");
    const bool dimacs = format == PSP_FORMAT_DIMACS;
    try {
        return finish_graph(parse_graph_device(t, dimacs, name, ctx->stream, ctx->sms));
    } catch (const GraphError& e) {
        // psp::Graph(n, edges) failing on an edge list surfaces as a
        // ParseError at the last line (src/graph_io.cpp:88-93); normalised
        // DIMACS input cannot fail it
        if (dimacs) throw;
        const uint64_t ln = count_lines(t);
        throw ParseFail{name + ":" + std::to_string(ln) + ": " + e.what(), ln};
    }
}
}  // namespace

psp_status psp_gpu_load_graph(psp_gpu_ctx* ctx, const char* path, int format, psp_graph** out) {
    return guarded([&] {
        if (!ctx || !path || !out) throw ArgError("load_graph: NULL argument");
        *out = nullptr;
        CK(cudaSetDevice(ctx->device));
        const auto t0 = Clock::now();
        DevText t;
        read_to_device(path, ctx->stream, t);
        CK(cudaStreamSynchronize(ctx->stream));
        const double read_ms = ms_since(t0);
        *out = parse_text(ctx, t, format, path);
        if (std::getenv("PSP_IO_PROFILE"))
            std::fprintf(stderr, "[load_graph] read+H2D %.1f ms, parse+validate %.1f ms\n", read_ms,
                         ms_since(t0) - read_ms);
    });
}

psp_status psp_gpu_read_graph(psp_gpu_ctx* ctx, const char* text, uint64_t len, int format,
                              const char* name, psp_graph** out) {
    return guarded([&] {
        if (!ctx || (!text && len) || !out) throw ArgError("read_graph: NULL argument");
        *out = nullptr;
        CK(cudaSetDevice(ctx->device));
        DevText t;
        text_to_device(text, len, ctx->stream, t);
        *out = parse_text(ctx, t, format, name ? name : "<stream>");
    });
}

psp_status psp_graph_size(const psp_graph* g, uint64_t* n, uint64_t* m) {
    return guarded([&] {
        if (!g) throw ArgError("graph_size: NULL graph");
        if (n) *n = g->n;
        if (m) *m = g->eu.size();
    });
}

psp_status psp_graph_edges(const psp_graph* g, uint32_t* eu, uint32_t* ev, double* ew) {
    return guarded([&] {
        if (!g) throw ArgError("graph_edges: NULL graph");
        if (eu) std::copy(g->eu.begin(), g->eu.end(), eu);
        if (ev) std::copy(g->ev.begin(), g->ev.end(), ev);
        if (ew) std::copy(g->ew.begin(), g->ew.end(), ew);
    });
}

void psp_graph_free(psp_graph* g) { delete g; }

uint64_t psp_gpu_last_parse_line(void) { return g_parse_line; }

psp_status psp_write_graph(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                           const double* ew, int format, char* buf, uint64_t cap, uint64_t* len) {
    return guarded([&] {
        if (m && (!eu || !ev || !ew)) throw ArgError("write_graph: NULL edge array");
        if (format != PSP_FORMAT_EDGE_LIST && format != PSP_FORMAT_DIMACS)
            throw ArgError("graph format must be PSP_FORMAT_EDGE_LIST or PSP_FORMAT_DIMACS");
        const Csr g = build_csr(n, m, eu, ev, ew);
        const std::string text = write_graph_text(g, format == PSP_FORMAT_DIMACS,
                                                  std::max(1u, std::thread::hardware_concurrency()));
        if (len) *len = text.size();
        if (buf) {
            if (cap < text.size()) throw ArgError("write_graph: buffer too small");
            std::memcpy(buf, text.data(), text.size());
        }
    });
}

psp_status psp_save_graph(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                          const double* ew, const char* path, int format) {
    return guarded([&] {
        if (!path) throw ArgError("save_graph: NULL path");
        if (m && (!eu || !ev || !ew)) throw ArgError("save_graph: NULL edge array");
        if (format != PSP_FORMAT_EDGE_LIST && format != PSP_FORMAT_DIMACS)
            throw ArgError("graph format must be PSP_FORMAT_EDGE_LIST or PSP_FORMAT_DIMACS");
        const Csr g = build_csr(n, m, eu, ev, ew);
        const std::string text = write_graph_text(g, format == PSP_FORMAT_DIMACS,
                                                  std::max(1u, std::thread::hardware_concurrency()));
        std::ofstream f(path, std::ios::binary);
        if (!f) throw Fail{PSP_EIO, std::string("cannot open '") + path + "' for writing"};
        f.write(text.data(), std::streamsize(text.size()));
        f.flush();
        if (!f) throw Fail{PSP_EIO, std::string("write to '") + path + "' failed"};
    });
}

uint32_t psp_format_weight(double w, char* buf) { return buf ? format_weight_into(w, buf) : 0; }

psp_status psp_gpu_minplus_peak(psp_gpu_ctx* ctx, int value_kind, double* relax_per_s,
                                double* sm_clock_mhz) {
    return guarded([&] {
        if (!ctx || !relax_per_s) throw ArgError("minplus_peak: NULL argument");
        CK(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        DBuf out(ctx->sms * 64 * sizeof(uint32_t));
        const int blocks = ctx->sms * 4;
        const uint32_t iters = 1 << 13;
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
        *relax_per_s = double(blocks) * NTHREADS * 128.0 * iters / (ms * 1e-3);
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

psp_status psp_min_spanning_forest(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                                   const double* key, uint8_t* in_tree) {
    return guarded([&] {
        if (m && (!eu || !ev || !key || !in_tree)) throw ArgError("min_spanning_forest: NULL argument");
        if (n > 0xffffffffull || m > 0xffffffffull) throw ArgError("min_spanning_forest: too large");
        for (uint64_t e = 0; e < m; ++e)
            if (eu[e] >= n || ev[e] >= n) throw ArgError("min_spanning_forest: vertex id out of range");
        min_spanning_forest(n, m, eu, ev, key, in_tree);
    });
}

psp_status psp_delaunay_edges(uint64_t n, const double* xy, uint64_t cap, uint32_t* eu,
                              uint32_t* ev, uint64_t* m) {
    return guarded([&] {
        if (!xy || !eu || !ev || !m) throw ArgError("delaunay_edges: NULL argument");
        std::vector<uint32_t> a, b;
        delaunay_edges(n, xy, a, b);
        if (a.size() > cap) throw ArgError("delaunay_edges: capacity too small");
        std::copy(a.begin(), a.end(), eu);
        std::copy(b.begin(), b.end(), ev);
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

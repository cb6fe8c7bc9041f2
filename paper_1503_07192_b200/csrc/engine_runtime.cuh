// engine_runtime.cuh — error plumbing, device buffers, tile arenas.
// Internal to libpsp_gpu.so (one translation unit: psp_gpu.cu includes the
// engine headers in dependency order).
#pragma once

namespace {

thread_local std::string g_err;
thread_local uint64_t g_parse_line = 0;  // psp::ParseError::line() of the last PSP_EPARSE

struct Fail {
    psp_status st;
    std::string msg;
};

struct ParseFail {  // psp::ParseError: "<name>:<line>: <msg>"
    std::string msg;
    uint64_t line;
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
    } catch (const ParseFail& e) {
        g_err = e.msg;
        g_parse_line = e.line;
        return PSP_EPARSE;
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
// Freed buffers up to kMaxBuf bytes are kept for reuse (at most kMaxHeld
// bytes per process). On these boxes a cudaMalloc/cudaFree pair costs 1-9 ms
// and single calls have stalled for up to 0.85 s (profiles/r1s5_component_laps),
// and a build makes hundreds of small ones (uploads, arena metadata, lists).
// Semantics kept from cudaFree: the give-back synchronizes the device first,
// so a cached block is idle when it is handed out again. Budgets count cached
// bytes as free (mem_info), and an allocation that fails flushes and retries,
// so budget decisions and OOM behaviour are what they were without it.
class BufCache {
public:
    static constexpr size_t kMaxBuf = size_t(64) << 20, kMaxHeld = size_t(1) << 30;
    static size_t rounded(size_t n) {
        if (n <= (size_t(1) << 20)) {
            size_t r = 256;
            while (r < n) r <<= 1;
            return r;
        }
        const size_t g = size_t(2) << 20;
        return (n + g - 1) / g * g;
    }
    void* take(size_t n) {
        if (n > kMaxBuf || off_) return nullptr;
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu_);
        auto it = free_.find({dev, rounded(n)});
        if (it == free_.end()) return nullptr;
        void* p = it->second;
        held_ -= it->first.second;
        free_.erase(it);
        return p;
    }
    bool give(void* p, size_t n) {
        if (n > kMaxBuf || off_) return false;
        // file the block under the device that owns it, not the current one
        // (a pipe or oracle may be released from another device's thread)
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
            cudaGetLastError();
            return false;
        }
        const int dev = at.device;
        const size_t r = rounded(n);
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (held_ + r > kMaxHeld) return false;
        }
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        const bool idle = cudaDeviceSynchronize() == cudaSuccess;  // as cudaFree would
        if (cur != dev) cudaSetDevice(cur);
        if (!idle) return false;
        std::lock_guard<std::mutex> lk(mu_);
        if (held_ + r > kMaxHeld) return false;  // another thread filled the cache meanwhile
        free_.emplace(std::make_pair(dev, r), p);
        held_ += r;
        return true;
    }
    size_t held() {
        std::lock_guard<std::mutex> lk(mu_);
        return held_;
    }
    void flush() {
        std::lock_guard<std::mutex> lk(mu_);
        int cur = 0;
        cudaGetDevice(&cur);
        for (auto& [key, p] : free_) {
            if (key.first != cur) cudaSetDevice(key.first);
            cudaFree(p);
            if (key.first != cur) cudaSetDevice(cur);
        }
        free_.clear();
        held_ = 0;
    }

private:
    std::mutex mu_;
    std::multimap<std::pair<int, size_t>, void*> free_;
    size_t held_ = 0;
    const bool off_ = std::getenv("PSP_NO_BUF_CACHE") != nullptr;
};
BufCache& buf_cache() {
    static BufCache* c = new BufCache;  // never destroyed: frees after CUDA teardown are unsafe
    return *c;
}

// Large blocks (> BufCache::kMaxBuf) come from a per-device stream-ordered
// memory pool (cudaMallocFromPoolAsync) whose release threshold keeps freed
// memory reserved, so a build's arenas (tens of GB) are re-served without
// driver calls: on these boxes one cudaMalloc/cudaFree of that size costs
// milliseconds and single calls have stalled for up to 0.8 s in the middle of
// a build. Semantics stay cudaMalloc/cudaFree's: the allocation is complete
// before it is handed out (its stream is synchronised), a free first
// synchronises the device, and reserved-but-unused pool memory counts as free
// (mem_info), trimmed when the real free memory runs low or an allocation
// fails. IPC-exported buffers (DBuf::alloc_ipc) bypass the pool.
// OFF by default: measured on cfg3 it made builds slower, not steadier
// (boundary phase minus K2 0.10-0.82 s with cudaMalloc, 6.4-17 s with the
// pool: growing a pool by tens of GB in the middle of a build and trimming it
// when the real free memory runs low cost far more than the calls it saves;
// profiles/r2/build_repeat_cfg3_{nopool,pool}.jsonl). PSP_POOL=1 turns it on.
class BigPool {
public:
    static constexpr int kMaxDev = 64;
    bool enabled() const { return !off_; }
    void* take(size_t n) {
        if (off_) return nullptr;
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= kMaxDev) return nullptr;
        Dev& d = get(dev);
        if (!d.pool) return nullptr;
        void* p = nullptr;
        cudaError_t e = cudaMallocFromPoolAsync(&p, n, d.pool, d.stream);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            cudaDeviceSynchronize();
            cudaMemPoolTrimTo(d.pool, 0);
            e = cudaMallocFromPoolAsync(&p, n, d.pool, d.stream);
        }
        if (e != cudaSuccess) {
            cudaGetLastError();
            return nullptr;  // the caller falls back to cudaMalloc (and its errors)
        }
        if (cudaStreamSynchronize(d.stream) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return p;
    }
    void give(void* p) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) == cudaSuccess) dev = at.device;
        cudaGetLastError();
        int cur = dev;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        cudaDeviceSynchronize();  // as cudaFree would
        cudaFreeAsync(p, get(dev).stream);
        if (cur != dev) cudaSetDevice(cur);
    }
    // reserved-but-unused bytes of the current device's pool
    size_t idle() {
        if (off_) return 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= kMaxDev || !devs_[dev].pool) return 0;
        uint64_t res = 0, used = 0;
        cudaMemPoolGetAttribute(devs_[dev].pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(devs_[dev].pool, cudaMemPoolAttrUsedMemCurrent, &used);
        return res > used ? size_t(res - used) : 0;
    }
    void trim() {
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= kMaxDev || !devs_[dev].pool) return;
        cudaStreamSynchronize(devs_[dev].stream);
        cudaMemPoolTrimTo(devs_[dev].pool, 0);
    }

private:
    struct Dev {
        cudaMemPool_t pool = nullptr;
        cudaStream_t stream = nullptr;
        bool tried = false;
    };
    Dev& get(int dev) {
        std::lock_guard<std::mutex> lk(mu_);
        Dev& d = devs_[dev];
        if (!d.tried) {
            d.tried = true;
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            if (cudaMemPoolCreate(&d.pool, &props) == cudaSuccess) {
                uint64_t keep = ~0ull;
                cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &keep);
                if (cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking) != cudaSuccess)
                    d.pool = nullptr;
            } else {
                d.pool = nullptr;
            }
            cudaGetLastError();
        }
        return d;
    }
    std::mutex mu_;
    Dev devs_[kMaxDev];
    const bool off_ = std::getenv("PSP_POOL") == nullptr;
};
BigPool& big_pool() {
    static BigPool* p = new BigPool;  // never destroyed (see buf_cache)
    return *p;
}
// free device memory as the budgets see it: cached blocks count as free
// (flushing them here costs 0.4-0.7 s of cudaFree on these boxes); a large
// allocation that then does not fit flushes the cache and retries (DBuf::alloc)
// But memory taken outside DBuf (NCCL buffers, lazy module loads, local-memory
// resizes) cannot use cached blocks: when the real free memory drops under
// kFlushBelow (the callers' margins are 1-2 GB), the cache is flushed first.
void mem_info(size_t* free_b, size_t* total_b) {
    constexpr size_t kFlushBelow = size_t(2) << 30;
    CK(cudaMemGetInfo(free_b, total_b));
    if (*free_b < kFlushBelow && (buf_cache().held() > 0 || big_pool().idle() > 0)) {
        buf_cache().flush();
        big_pool().trim();
        CK(cudaMemGetInfo(free_b, total_b));
    }
    *free_b += buf_cache().held() + big_pool().idle();
}

// Host time spent inside cudaMalloc / cudaFree of device buffers (process
// totals, psp_gpu_alloc_stats): on these boxes single calls have stalled for
// 0.1-1 s, which is most of the build's wall-clock noise.
std::atomic<uint64_t> g_malloc_ns{0}, g_free_ns{0}, g_malloc_calls{0}, g_free_calls{0};
struct AllocTimer {
    std::atomic<uint64_t>& ns;
    size_t bytes = 0;
    const char* what = "";
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~AllocTimer() {
        const uint64_t d = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                        std::chrono::steady_clock::now() - t0).count());
        ns += d;
        static const bool log = std::getenv("PSP_ALLOC_LOG") != nullptr;  // calls over 2 ms
        if (log && d > 2000000)
            std::fprintf(stderr, "[psp] %s of %.3f GB took %.1f ms\n", what, bytes / 1e9, d / 1e6);
    }
};

struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    bool pooled = false, ipc = false;
    bool borrowed = false;  // a view into another buffer: never freed here
    DBuf() = default;
    explicit DBuf(size_t n) { alloc(n); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes), pooled(o.pooled), ipc(o.ipc), borrowed(o.borrowed) {
        o.p = nullptr;
        o.bytes = 0;
        o.pooled = o.ipc = o.borrowed = false;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p;
            bytes = o.bytes;
            pooled = o.pooled;
            ipc = o.ipc;
            borrowed = o.borrowed;
            o.p = nullptr;
            o.bytes = 0;
            o.pooled = o.ipc = o.borrowed = false;
        }
        return *this;
    }
    void borrow(void* at, size_t n) {
        reset();
        p = at;
        bytes = n;
        borrowed = true;
    }
    ~DBuf() { reset(); }
    void alloc(size_t n) {
        reset();
        if (n == 0) n = 16;
        bytes = n;
        if ((p = buf_cache().take(n))) return;
        if (n > BufCache::kMaxBuf && (p = big_pool().take(n))) {
            pooled = true;
            return;
        }
        const size_t r = n <= BufCache::kMaxBuf ? BufCache::rounded(n) : n;
        cudaError_t e;
        {
            AllocTimer t{g_malloc_ns, r, "cudaMalloc"};
            ++g_malloc_calls;
            e = cudaMalloc(&p, r);
            if (e == cudaErrorMemoryAllocation) {
                cudaGetLastError();
                buf_cache().flush();
                e = cudaMalloc(&p, r);
            }
        }
        if (e != cudaSuccess) {
            p = nullptr;
            bytes = 0;
            CK(e);
        }
    }
    // a plain cudaMalloc block (neither cached nor pooled): CUDA IPC
    // handles (cudaIpcGetMemHandle) need one
    void alloc_ipc(size_t n) {
        reset();
        if (n == 0) n = 16;
        bytes = n;
        ipc = true;
        CK(cudaMalloc(&p, n));
    }
    void reset() {
        if (p && !borrowed) {
            if (pooled) {
                big_pool().give(p);
            } else if (ipc || !buf_cache().give(p, bytes)) {
                AllocTimer t{g_free_ns, bytes, "cudaFree"};
                ++g_free_calls;
                cudaFree(p);
            }
        }
        p = nullptr;
        bytes = 0;
        pooled = ipc = borrowed = false;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

template <class T>
DBuf upload(const std::vector<T>& h, cudaStream_t s) {
    DBuf d(h.size() * sizeof(T));
    if (!h.empty()) CK(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
}

// Bulk copy between device memory and PAGEABLE host memory at PCIe speed:
// worker threads each stage 64 MB chunks through their own pinned buffer and
// stream (pageable cudaMemcpy runs at a few GB/s; pinning tens of GB up
// front costs more than the copy).
inline void staged_copy(void* dst, const void* src, size_t bytes, bool to_host, int device) {
    const size_t chunk = 64ull << 20;
    const size_t nchunks = (bytes + chunk - 1) / chunk;
    const unsigned nthreads =
        static_cast<unsigned>(std::min<size_t>(nchunks, std::max(2u, std::min(8u, std::thread::hardware_concurrency()))));
    std::vector<std::thread> pool;
    std::vector<Fail> fails(nthreads, Fail{PSP_OK, ""});
    for (unsigned t = 0; t < nthreads; ++t) {
        pool.emplace_back([&, t] {
            void* pin = nullptr;
            cudaStream_t st = nullptr;
            try {
                CK(cudaSetDevice(device));
                CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
                CK(cudaMallocHost(&pin, chunk));
                for (size_t c = t; c < nchunks; c += nthreads) {
                    const size_t off = c * chunk, len = std::min(chunk, bytes - off);
                    if (to_host) {
                        CK(cudaMemcpyAsync(pin, static_cast<const char*>(src) + off, len,
                                           cudaMemcpyDeviceToHost, st));
                        CK(cudaStreamSynchronize(st));
                        std::memcpy(static_cast<char*>(dst) + off, pin, len);
                    } else {
                        std::memcpy(pin, static_cast<const char*>(src) + off, len);
                        CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, pin, len,
                                           cudaMemcpyHostToDevice, st));
                        CK(cudaStreamSynchronize(st));
                    }
                }
            } catch (const Fail& f) {
                fails[t] = f;
            }
            if (pin) cudaFreeHost(pin);
            if (st) cudaStreamDestroy(st);
        });
    }
    for (auto& th : pool) th.join();
    for (auto& f : fails)
        if (f.st != PSP_OK) throw f;
}

// ------------------------------------------------- partially backed range --
// One contiguous virtual range of which only chosen byte ranges own device
// memory (CUDA virtual memory management; driver entry points fetched through
// the runtime, no -lcuda). The rest maps, in pieces, onto one small shared
// "sink" allocation: kernels may then address the whole range as one array
// and write anywhere (initialisation passes that sweep every tile), while
// only the backed ranges hold data. Readers must stay inside backed ranges.
// Used for the row-sharded boundary-graph table (PSP_STORAGE_ROW_SHARDED):
// rank r backs the tile rows it owns, about 1/world of the table.
struct VmmApi {
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    bool ok = false;
};
const VmmApi& vmm_api() {
    static VmmApi a = [] {
        VmmApi v;
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q{};
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn;
        };
        v.ok = get("cuMemAddressReserve", reinterpret_cast<void**>(&v.reserve)) &&
               get("cuMemAddressFree", reinterpret_cast<void**>(&v.addr_free)) &&
               get("cuMemCreate", reinterpret_cast<void**>(&v.create)) &&
               get("cuMemRelease", reinterpret_cast<void**>(&v.release)) &&
               get("cuMemMap", reinterpret_cast<void**>(&v.map)) &&
               get("cuMemUnmap", reinterpret_cast<void**>(&v.unmap)) &&
               get("cuMemSetAccess", reinterpret_cast<void**>(&v.set_access)) &&
               get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&v.granularity));
        cudaGetLastError();
        return v;
    }();
    return a;
}

struct PartialRange {
    CUdeviceptr va = 0;
    size_t size = 0, gran = 0, backed = 0, sink_bytes = 0;
    std::vector<std::pair<size_t, size_t>> maps;   // (offset, length) of every mapping
    std::vector<std::pair<size_t, size_t>> owned;  // backed byte ranges (granule-aligned)
    // cuMemMap maps whole allocations only (offset 0, full size): one
    // allocation per backed run, and sinks of power-of-two granule counts,
    // each mapped wherever a piece of its size falls in the unbacked gaps
    std::vector<CUmemGenericAllocationHandle> runs;
    std::map<size_t, CUmemGenericAllocationHandle> sinks;

    PartialRange() = default;
    PartialRange(const PartialRange&) = delete;
    PartialRange& operator=(const PartialRange&) = delete;
    ~PartialRange() { reset(); }

    static void dck(CUresult r, const char* what) {
        if (r != CUDA_SUCCESS)
            throw Fail{r == CUDA_ERROR_OUT_OF_MEMORY ? PSP_ENOMEM : PSP_ECUDA,
                       std::string(what) + " failed (CUresult " + std::to_string(int(r)) + ")"};
    }
    // `want`: byte ranges that must hold data (any order, may overlap)
    void create(int device, size_t bytes, std::vector<std::pair<size_t, size_t>> want) {
        reset();
        const VmmApi& api = vmm_api();
        if (!api.ok) throw Fail{PSP_ECUDA, "CUDA virtual memory management entry points unavailable"};
        CUmemAllocationProp prop{};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = device;
        dck(api.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
        size = std::max(gran, (bytes + gran - 1) / gran * gran);
        // granule-aligned, merged ranges
        for (auto& w : want) {
            const size_t a = w.first / gran * gran;
            const size_t b = std::min(size, (w.first + w.second + gran - 1) / gran * gran);
            if (b > a) owned.emplace_back(a, b - a);
        }
        std::sort(owned.begin(), owned.end());
        std::vector<std::pair<size_t, size_t>> merged;
        for (auto& r : owned) {
            if (!merged.empty() && r.first <= merged.back().first + merged.back().second)
                merged.back().second = std::max(merged.back().first + merged.back().second,
                                                r.first + r.second) - merged.back().first;
            else merged.push_back(r);
        }
        owned.swap(merged);
        for (auto& r : owned) backed += r.second;
        const size_t max_sink = std::max(gran, size_t(64) << 20);
        try {
            dck(api.reserve(&va, size, gran, 0, 0), "cuMemAddressReserve");
            auto map_sink = [&](size_t from, size_t to) {
                for (size_t o = from; o < to;) {
                    size_t len = gran;  // largest power-of-two granule count that fits
                    while (len * 2 <= std::min(max_sink, to - o)) len *= 2;
                    auto it = sinks.find(len);
                    if (it == sinks.end()) {
                        CUmemGenericAllocationHandle h = 0;
                        dck(api.create(&h, len, &prop, 0), "cuMemCreate(sink)");
                        it = sinks.emplace(len, h).first;
                        sink_bytes += len;
                    }
                    dck(api.map(va + o, len, 0, it->second, 0), "cuMemMap(sink)");
                    maps.emplace_back(o, len);
                    o += len;
                }
            };
            size_t at = 0;
            for (auto& r : owned) {
                map_sink(at, r.first);
                CUmemGenericAllocationHandle h = 0;
                dck(api.create(&h, r.second, &prop, 0), "cuMemCreate(table rows)");
                runs.push_back(h);
                dck(api.map(va + r.first, r.second, 0, h, 0), "cuMemMap(rows)");
                maps.emplace_back(r.first, r.second);
                at = r.first + r.second;
            }
            map_sink(at, size);
            CUmemAccessDesc acc{};
            acc.location = prop.location;
            acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            dck(api.set_access(va, size, &acc, 1), "cuMemSetAccess");
        } catch (...) {
            reset();
            throw;
        }
    }
    void reset() {
        const VmmApi& api = vmm_api();
        if (va) {
            cudaDeviceSynchronize();  // as cudaFree would
            for (auto& m : maps) api.unmap(va + m.first, m.second);
            api.addr_free(va, size);
        }
        for (auto h : runs) api.release(h);
        for (auto& kv : sinks) api.release(kv.second);
        va = 0;
        runs.clear();
        sinks.clear();
        size = backed = sink_bytes = 0;
        maps.clear();
        owned.clear();
    }
    void* ptr() const { return reinterpret_cast<void*>(va); }
};

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
    // sparse walk (see MatSet::act_*): flags ride at the end of the panel
    // buffer (one per panel slot), the work lists in d_act; walked_tiles =
    // tile products actually executed (all phases, all ranks), read back
    // after the FW. PSP_FW_DENSE=1 walks every tile (A/B measurement).
    bool sparse = false;
    DBuf d_act;
    uint64_t walked_tiles = 0;
    uint64_t nslots = 0;  // sum of nb over the matrices (= panel slots)
    // row-sharded storage (a single matrix over `world` ranks): only the
    // tile rows I with I mod world == rank are backed by device memory
    std::unique_ptr<PartialRange> part;
    size_t min_tile_bytes = 0;  // tiles allocation at least this large (reused later)
    void* tiles_p() const { return part ? part->ptr() : tiles.p; }
    template <class V> V* tiles_as() const { return static_cast<V*>(tiles_p()); }

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

    // sparse_walk: -1 = the default (a single matrix, i.e. the boundary
    // graph), 0 / 1 = off / on for a batch of matrices
    // row_shard = {device, rank, world}: back only this rank's tile rows
    // (nmat == 1, see PartialRange); nullptr = one ordinary allocation
    void create(const std::vector<uint64_t>& sizes, size_t value_bytes, bool with_panel,
                cudaStream_t s, int sparse_walk = -1, const int* row_shard = nullptr) {
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
        nslots = panel_elems / TT;
        part.reset();
        tiles.reset();
        if (row_shard && nmat == 1) {
            const uint32_t r = uint32_t(row_shard[1]), g = uint32_t(row_shard[2]);
            std::vector<std::pair<size_t, size_t>> rows;
            for (uint32_t I = r; I < nb[0]; I += g)
                rows.emplace_back(tidx(I, I, nb[0]) * TT * vbytes, uint64_t(nb[0] - I) * TT * vbytes);
            part = std::make_unique<PartialRange>();
            part->create(row_shard[0], tile_elems * vbytes, rows);
        } else {
            tiles.alloc(std::max<size_t>(tile_elems * vbytes, min_tile_bytes));
        }
        sparse = with_panel && nb_max > 1 && std::getenv("PSP_FW_DENSE") == nullptr &&
                 (sparse_walk < 0 ? nmat == 1 : sparse_walk > 0);
        const size_t panel_bytes = (panel_elems + (sparse ? nslots : 0)) * vbytes;
        const size_t tail = (tile_elems * vbytes + 255) / 256 * 256;
        if (with_panel && !part && tail + panel_bytes <= tiles.bytes)
            panel.borrow(static_cast<char*>(tiles.p) + tail, panel_bytes);  // spare room of a larger allocation
        else if (with_panel) panel.alloc(panel_bytes);
        if (sparse) d_act.alloc(act_bytes());
        d_tile_base = upload(tile_base, s);
        d_panel_base = upload(panel_base, s);
        d_work_prefix = upload(work_prefix, s);
        d_nb = upload(nb, s);
    }
    template <class V> MatSet<V> view() const {
        MatSet<V> v;
        v.tiles = tiles_as<V>();
        v.diag = nullptr;
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
        v.p2p = 0;
        const bool sp = sparse && panel.p && d_act.p;
        v.act_flag = sp ? panel.as<V>() + panel_elems : nullptr;
        unsigned char* ab = sp ? d_act.as<unsigned char>() : nullptr;
        // d_act: act_work | act_prefix (nslots + nmat) | mat_prefix (nmat + 1)
        //        | act_list (nslots) | act_rows (nslots) | act_meta (2 nmat)
        v.act_work = sp ? reinterpret_cast<unsigned long long*>(ab) : nullptr;
        v.act_prefix = sp ? reinterpret_cast<uint64_t*>(ab + 8) : nullptr;
        v.mat_prefix = sp ? v.act_prefix + nslots + nmat : nullptr;
        v.act_list = sp ? reinterpret_cast<uint32_t*>(v.mat_prefix + nmat + 1) : nullptr;
        v.act_rows = sp ? v.act_list + nslots : nullptr;
        v.act_meta = sp ? v.act_rows + nslots : nullptr;
        return v;
    }
    size_t act_bytes() const { return 8 * (1 + nslots + 2 * uint64_t(nmat) + 1) + 4 * (2 * nslots + 2 * uint64_t(nmat)); }
    unsigned long long* act_work_ptr() const { return reinterpret_cast<unsigned long long*>(d_act.p); }
    // relaxations the FW executes on the padded matrices: per k-block the
    // diagonal tile, the nb-1 panel tiles and the upper tiles off row/col kb
    uint64_t relaxations() const {
        if (sparse)  // diagonal, computed panel and walked phase-3 tiles
            return walked_tiles * uint64_t(T) * T * T;
        uint64_t r = 0;
        for (uint32_t m = 0; m < nmat; ++m) r += ntiles_upper(nb[m]) * nb[m];
        return r * uint64_t(T) * T * T;
    }
    size_t bytes() const {
        return (part ? part->backed + part->sink_bytes : tiles.bytes) + panel.bytes;
    }
    // backed byte ranges of the tile storage (all of it when not row-sharded)
    std::vector<std::pair<size_t, size_t>> backed_ranges() const {
        if (part) return part->owned;
        return {{0, tile_elems * vbytes}};
    }
};

}  // namespace


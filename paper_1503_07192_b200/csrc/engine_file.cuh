// engine_file.cuh — PSP1 oracle files from/to device tables (host side).
// Internal to libpsp_gpu.so (one translation unit: psp_gpu.cu includes the
// engine headers in dependency order).
#pragma once

// --------------------------------------------------------- PSP1 files --
struct PinnedBuf {
    void* p = nullptr;
    explicit PinnedBuf(size_t n) { CK(cudaMallocHost(&p, n)); }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

constexpr size_t IO_CHUNK = size_t(64) << 20;  // bytes per device/host staging chunk

// GPU side of the running CRC: the slicing tables and the fold matrices
// (crc64_blocks), set up once per call site.
struct GpuCrc {
    DBuf slices, out;
    std::vector<uint64_t> hout;
    explicit GpuCrc(const Crc64Stream& crc, cudaStream_t s) {
        static const Crc64Slices sl = make_crc64_slices();
        slices.alloc(sizeof(Crc64Slices));
        CK(cudaMemcpyAsync(slices.p, &sl, sizeof sl, cudaMemcpyHostToDevice, s));
        CrcFold fold;
        for (int j = 0; j < 8; ++j)
            for (int b = 0; b < 64; ++b) fold.col[j][b] = crc.shift_pow2(8 + j).col[b];
        CK(cudaMemcpyToSymbolAsync(c_crc_fold, &fold, sizeof fold, 0, cudaMemcpyHostToDevice, s));
        static bool attr = false;
        if (!attr) {
            CK(cudaFuncSetAttribute(crc64_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(8 * 256 * 8 + CRC_BLOCK)));
            attr = true;
        }
    }
    // raw CRCs of the full 64 KB blocks of d[0, len) (enqueued on s; read
    // with fold() after the stream is synchronised)
    uint64_t launch(const uint8_t* d, uint64_t len, cudaStream_t s) {
        const uint64_t nblk = len / CRC_BLOCK;
        if (nblk == 0) return 0;
        if (out.bytes < nblk * 8) out.alloc(nblk * 8);
        hout.resize(nblk);
        crc64_blocks<<<unsigned(nblk), CRC_THREADS, 8 * 256 * 8 + CRC_BLOCK, s>>>(
            d, slices.as<Crc64Slices>(), out.as<uint64_t>());
        CK_LAUNCH();
        CK(cudaMemcpyAsync(hout.data(), out.p, nblk * 8, cudaMemcpyDeviceToHost, s));
        return nblk;
    }
    // append the blocks, then the sub-block tail from the host copy `h`
    void fold(Crc64Stream& crc, uint64_t nblk, const uint8_t* h, uint64_t len) {
        for (uint64_t i = 0; i < nblk; ++i) crc.append_raw(hout[i], CRC_BLOCK);
        crc.update(h + nblk * CRC_BLOCK, len - nblk * CRC_BLOCK);
    }
};

inline void pwrite_all(int fd, const void* src, uint64_t len, uint64_t off) {
    constexpr int kThreads = 8;
    const uint64_t per = (len + kThreads - 1) / kThreads;
    std::atomic<bool> failed{false};
    std::vector<std::thread> th;
    for (int t = 0; t < kThreads; ++t) {
        const uint64_t a = std::min(len, t * per), b = std::min(len, a + per);
        if (a >= b) break;
        th.emplace_back([&, a, b] {
            for (uint64_t at = a; at < b && !failed;) {
                const ssize_t r = ::pwrite(fd, static_cast<const char*>(src) + at, b - at, off + at);
                if (r <= 0) failed = true;
                else at += uint64_t(r);
            }
        });
    }
    for (auto& x : th) x.join();
    if (failed) throw Fail{PSP_EIO, "oracle write failed"};
}

// Tables in file order (component tables, then boundary rows), converted to
// f64 on the device into a 64 MB staging chunk (windows packed back to
// back), CRC'd on the device, copied to pinned host memory and written with
// parallel pwrites at `off`; the write of one chunk overlaps the device work
// of the next (two staging buffers, one write in flight). Returns the end
// offset.
template <class V>
uint64_t save_tables(const psp_gpu_oracle* o, int fd, uint64_t off, Crc64Stream& crc) {
    cudaStream_t s = o->ctx->stream;
    DBuf chunk[2] = {DBuf(IO_CHUNK), DBuf(IO_CHUNK)};
    PinnedBuf host[2] = {PinnedBuf(IO_CHUNK), PinnedBuf(IO_CHUNK)};
    GpuCrc gcrc(crc, s);
    std::future<void> writing;
    int cur = 0;
    uint64_t fill = 0;  // bytes staged in chunk[cur]
    auto finish_write = [&] {
        if (writing.valid()) writing.get();  // rethrows a write failure
    };
    auto flush = [&] {
        if (!fill) return;
        const uint64_t nblk = gcrc.launch(chunk[cur].as<uint8_t>(), fill, s);
        CK(cudaMemcpyAsync(host[cur].p, chunk[cur].p, fill, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint8_t* h = static_cast<const uint8_t*>(host[cur].p);
        gcrc.fold(crc, nblk, h, fill);
        finish_write();  // the previous chunk (the other buffer)
        writing = std::async(std::launch::async, [fd, h, len = fill, at = off] { pwrite_all(fd, h, len, at); });
        off += fill;
        fill = 0;
        cur ^= 1;
    };
    auto emit = [&](const MatArena& a, uint32_t m, uint32_t row0, uint32_t nrows, uint32_t ncols) {
        if (!nrows || !ncols) return;
        const uint64_t row_bytes = uint64_t(ncols) * 8;
        if (row_bytes > IO_CHUNK) throw Fail{PSP_EINVAL, "oracle_save: rows longer than 8M entries"};
        for (uint32_t r0 = 0; r0 < nrows;) {
            const uint64_t room = (IO_CHUNK - fill) / row_bytes;
            if (room == 0) {
                flush();
                continue;
            }
            const uint32_t nr = uint32_t(std::min<uint64_t>(room, nrows - r0));
            const uint64_t cnt = uint64_t(nr) * ncols;
            window_to_f64<V><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(
                a.view<V>(), m, row0 + r0, nr, ncols, o->scale,
                reinterpret_cast<double*>(chunk[cur].as<uint8_t>() + fill));
            CK_LAUNCH();
            fill += cnt * 8;
            r0 += nr;
        }
    };
    const Reordered& R = o->R;
    for (uint32_t c = 0; c < R.k; ++c) {
        const uint32_t sz = R.comp_off[c + 1] - R.comp_off[c];
        emit(o->comps, c, 0, sz, sz);
    }
    for (uint32_t c = 0; c < R.k; ++c)
        emit(o->bg, 0, R.bnd_off[c], R.bnd_off[c + 1] - R.bnd_off[c], uint32_t(R.b()));
    flush();
    finish_write();
    return off;
}

void put_u64s(std::vector<uint8_t>& buf, uint64_t v) {
    const size_t at = buf.size();
    buf.resize(at + 8);
    std::memcpy(buf.data() + at, &v, 8);
}


// ---- PSP1 load: the table section streamed from the file to the device.
// Chunks of IO_CHUNK bytes are read with parallel preads into pinned buffers
// (the read of chunk i + 1 overlaps the device work of chunk i), copied to
// HBM, CRC'd there (crc64_blocks) and converted straight into the tile-packed
// arenas (psp1_convert), which also reports the largest finite value and the
// fixed-point need for the value-kind decision. `crc` (if given) continues
// over the section.
struct Psp1Analysis {
    double maxv = 0.0;
    int need_q = 0;
};

inline void pread_all(int fd, void* dst, uint64_t len, uint64_t off, const std::string& name) {
    constexpr int kThreads = 8;
    const uint64_t per = (len + kThreads - 1) / kThreads;
    std::atomic<bool> failed{false};
    std::vector<std::thread> th;
    for (int t = 0; t < kThreads; ++t) {
        const uint64_t a = std::min(len, t * per), b = std::min(len, a + per);
        if (a >= b) break;
        th.emplace_back([&, a, b] {
            for (uint64_t at = a; at < b && !failed;) {
                const ssize_t r = ::pread(fd, static_cast<char*>(dst) + at, b - at, off + at);
                if (r <= 0) failed = true;
                else at += uint64_t(r);
            }
        });
    }
    for (auto& x : th) x.join();
    if (failed) throw Fail{PSP_EIO, name + ": truncated oracle file"};
}

template <class V>
Psp1Analysis stream_psp1_tables(psp_gpu_oracle* o, int fd, const std::string& name, uint64_t table_at,
                                uint64_t table_bytes, int shift, Crc64Stream* crc) {
    psp_gpu_ctx* ctx = o->ctx;
    cudaStream_t s = ctx->stream;
    const Reordered& R = o->R;
    const uint32_t k = R.k;
    const uint64_t b = R.b();
    // piece map in elements, file order
    std::vector<uint64_t> start(2 * size_t(k) + 1, 0);
    std::vector<uint32_t> size(k);
    for (uint32_t c = 0; c < k; ++c) {
        size[c] = R.comp_off[c + 1] - R.comp_off[c];
        start[c + 1] = start[c] + uint64_t(size[c]) * size[c];
    }
    for (uint32_t c = 0; c < k; ++c)
        start[k + c + 1] = start[k + c] + uint64_t(R.bnd_off[c + 1] - R.bnd_off[c]) * b;
    DBuf d_start = upload(start, s), d_size = upload(size, s), d_bnd = upload(R.bnd_off, s);
    const Psp1Map map{d_start.as<uint64_t>(), d_size.as<uint32_t>(), d_bnd.as<uint32_t>(), k,
                      static_cast<uint32_t>(b)};
    DBuf stats(16);
    CK(cudaMemsetAsync(stats.p, 0, 16, s));
    auto* d_max = stats.as<unsigned long long>();
    int* d_need = reinterpret_cast<int*>(stats.as<unsigned long long>() + 1);
    const MatSet<V> cv = o->comps.view<V>();
    const MatSet<V> bv = o->bg.nmat ? o->bg.view<V>() : MatSet<V>{};
    constexpr int PER = 8;
    PinnedBuf host[2] = {PinnedBuf(IO_CHUNK), PinnedBuf(IO_CHUNK)};
    DBuf dev[2] = {DBuf(IO_CHUNK), DBuf(IO_CHUNK)};
    cudaEvent_t done[2];
    for (auto& e : done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct Ev {
        cudaEvent_t* e;
        ~Ev() {
            cudaEventDestroy(e[0]);
            cudaEventDestroy(e[1]);
        }
    } ev_guard{done};
    std::unique_ptr<GpuCrc> gcrc[2];
    if (crc)
        for (auto& g : gcrc) g = std::make_unique<GpuCrc>(*crc, s);
    uint64_t pending_nblk[2] = {0, 0}, pending_len[2] = {0, 0};
    bool busy[2] = {false, false};
    auto retire = [&](int slot) {  // the slot's device work is complete: fold its CRC
        if (!busy[slot]) return;
        CK(cudaEventSynchronize(done[slot]));
        if (crc) gcrc[slot]->fold(*crc, pending_nblk[slot], static_cast<const uint8_t*>(host[slot].p),
                                  pending_len[slot]);
        busy[slot] = false;
    };
    const uint64_t nchunks = (table_bytes + IO_CHUNK - 1) / IO_CHUNK;
    for (uint64_t ci = 0; ci < nchunks; ++ci) {
        const int slot = int(ci & 1);
        retire(slot);  // its pinned buffer and device chunk are free again
        const uint64_t at = ci * IO_CHUNK, len = std::min<uint64_t>(IO_CHUNK, table_bytes - at);
        pread_all(fd, host[slot].p, len, table_at + at, name);
        CK(cudaMemcpyAsync(dev[slot].p, host[slot].p, len, cudaMemcpyHostToDevice, s));
        if (crc) pending_nblk[slot] = gcrc[slot]->launch(dev[slot].as<uint8_t>(), len, s);
        const uint64_t cnt = len / 8;
        const uint64_t threads = (cnt + PER - 1) / PER;
        if (cnt)
            psp1_convert<V, PER><<<unsigned((threads + 255) / 256), 256, 0, s>>>(
                dev[slot].as<double>(), at / 8, cnt, map, cv, bv, shift, d_max, d_need);
        CK_LAUNCH();
        CK(cudaEventRecord(done[slot], s));
        pending_len[slot] = len;
        busy[slot] = true;
    }
    // in file order: the older slot first
    if (nchunks >= 2) retire(int(nchunks & 1));
    retire(int((nchunks + 1) & 1));
    uint64_t h[2];
    CK(cudaMemcpyAsync(h, stats.p, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    Psp1Analysis a;
    std::memcpy(&a.maxv, &h[0], 8);
    a.need_q = static_cast<int>(h[1] & 0xffffffffu);
    return a;
}

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

// Tables in file order (component tables, then boundary rows), converted to
// f64 on the device window by window, CRC'd on the device, copied to pinned
// host memory and written; the fwrite of one window overlaps the device work
// of the next (two staging buffers, one write in flight).
template <class V>
void save_tables(const psp_gpu_oracle* o, std::FILE* f, Crc64Stream& crc) {
    cudaStream_t s = o->ctx->stream;
    DBuf chunk[2] = {DBuf(IO_CHUNK), DBuf(IO_CHUNK)};
    PinnedBuf host[2] = {PinnedBuf(IO_CHUNK), PinnedBuf(IO_CHUNK)};
    GpuCrc gcrc(crc, s);
    std::future<bool> writing;
    int cur = 0;
    auto finish_write = [&] {
        if (writing.valid() && !writing.get()) throw Fail{PSP_EIO, "oracle write failed"};
    };
    auto emit = [&](const MatArena& a, uint32_t m, uint32_t row0, uint32_t nrows, uint32_t ncols) {
        if (!nrows || !ncols) return;
        const uint32_t per = uint32_t(std::max<uint64_t>(1, IO_CHUNK / (uint64_t(ncols) * 8)));
        for (uint32_t r0 = 0; r0 < nrows; r0 += per) {
            const uint32_t nr = std::min(per, nrows - r0);
            const uint64_t cnt = uint64_t(nr) * ncols, bytes = cnt * 8;
            window_to_f64<V><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(
                a.view<V>(), m, row0 + r0, nr, ncols, o->scale, chunk[cur].as<double>());
            CK_LAUNCH();
            const uint64_t nblk = gcrc.launch(chunk[cur].as<uint8_t>(), bytes, s);
            CK(cudaMemcpyAsync(host[cur].p, chunk[cur].p, bytes, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const uint8_t* h = static_cast<const uint8_t*>(host[cur].p);
            gcrc.fold(crc, nblk, h, bytes);
            finish_write();  // the previous window (the other buffer)
            writing = std::async(std::launch::async,
                                 [f, h, bytes] { return std::fwrite(h, 1, bytes, f) == bytes; });
            cur ^= 1;
        }
    };
    const Reordered& R = o->R;
    for (uint32_t c = 0; c < R.k; ++c) {
        const uint32_t sz = R.comp_off[c + 1] - R.comp_off[c];
        emit(o->comps, c, 0, sz, sz);
    }
    for (uint32_t c = 0; c < R.k; ++c)
        emit(o->bg, 0, R.bnd_off[c], R.bnd_off[c + 1] - R.bnd_off[c], uint32_t(R.b()));
    finish_write();
}

void put_u64s(std::vector<uint8_t>& buf, uint64_t v) {
    const size_t at = buf.size();
    buf.resize(at + 8);
    std::memcpy(buf.data() + at, &v, 8);
}


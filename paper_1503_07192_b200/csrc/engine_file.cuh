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


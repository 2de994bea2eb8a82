// tpa_artifact_io.cuh -- the stranger artifact's file format (persistence.hpp,
// persistence.cpp:69-125) written from / read into device buffers, with the
// CRC-32 computed on the GPU (a C5 payload is 2.1 GB).
//
// Format (unchanged, little-endian): "TPA1", version u32 (1), n u64, c f64,
// eps f64, T u32, graph fingerprint u64, n x f64 scores, CRC-32 (IEEE,
// reflected 0xEDB88320, init / final 0xFFFFFFFF, persistence.cpp:16-32) of
// every prior byte.  48 + 8n bytes.
//
// GPU CRC-32: the CRC register update is linear over GF(2), so
//   crc(D) = raw(D) ^ M_|D|(0xFFFFFFFF) ^ 0xFFFFFFFF,
//   raw(A || B) = M_|B|(raw(A)) ^ raw(B),
// with raw() the register run from 0 and M_L the 32x32 operator "advance by L
// zero bytes" (zlib's crc32_combine construction).  One thread per 4 KiB chunk
// computes its raw CRC (table in shared memory); one thread per group of 256
// chunks folds them with M_4096; the host folds the groups.
// Included at the end of tpa_gpu.cu.
#pragma once

#include <cstdio>

namespace tpa {

constexpr uint32_t kCrcChunk = 4096, kCrcGroup = 256;

struct Gf2Mat {
    uint32_t col[32];  // image of bit j
};

__host__ __device__ inline uint32_t gf2_apply(const Gf2Mat& M, uint32_t v) {
    uint32_t r = 0;
    for (int j = 0; j < 32; ++j)
        if ((v >> j) & 1u) r ^= M.col[j];
    return r;
}

static Gf2Mat gf2_mul(const Gf2Mat& A, const Gf2Mat& B) {  // A after B
    Gf2Mat C;
    for (int j = 0; j < 32; ++j) C.col[j] = gf2_apply(A, B.col[j]);
    return C;
}

// M_L: the raw CRC register advanced over L zero bytes
static Gf2Mat crc_zeros_op(uint64_t len) {
    Gf2Mat bit;  // one zero bit, reflected polynomial
    bit.col[0] = 0xEDB88320u;
    for (int j = 1; j < 32; ++j) bit.col[j] = 1u << (j - 1);
    Gf2Mat byte = gf2_mul(bit, bit);
    byte = gf2_mul(byte, byte);
    byte = gf2_mul(byte, byte);  // 8 zero bits
    Gf2Mat M;
    for (int j = 0; j < 32; ++j) M.col[j] = 1u << j;
    Gf2Mat P = byte;
    while (len) {
        if (len & 1) M = gf2_mul(P, M);
        P = gf2_mul(P, P);
        len >>= 1;
    }
    return M;
}

static uint32_t crc_table_entry(uint32_t i) {
    uint32_t crc = i;
    for (int bit = 0; bit < 8; ++bit) crc = (crc >> 1) ^ ((crc & 1u) ? 0xEDB88320u : 0u);
    return crc;
}

__global__ void __launch_bounds__(256) k_crc_chunks(const uint8_t* __restrict__ data, uint64_t size,
                                                    const uint32_t* __restrict__ table, uint32_t* __restrict__ raw) {
    __shared__ uint32_t T[256];
    T[threadIdx.x] = table[threadIdx.x];
    __syncthreads();
    const uint64_t nch = (size + kCrcChunk - 1) / kCrcChunk;
    const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const uint64_t lo = c * kCrcChunk, hi = min(size, lo + kCrcChunk);
    uint32_t s = 0;
    uint64_t p = lo;
    for (; p + 16 <= hi; p += 16) {  // chunk starts are 16-byte aligned (the buffer is)
        const uint4 w = *reinterpret_cast<const uint4*>(data + p);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int b = 0; b < 4; ++b) s = T[(s ^ (ws[q] >> (8 * b))) & 0xffu] ^ (s >> 8);
    }
    for (; p < hi; ++p) s = T[(s ^ data[p]) & 0xffu] ^ (s >> 8);
    raw[c] = s;
}

__global__ void k_crc_fold(const uint32_t* __restrict__ raw, uint64_t nch, Gf2Mat M_chunk, Gf2Mat M_tail,
                           uint32_t* __restrict__ group_raw) {
    const uint64_t gidx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t lo = gidx * kCrcGroup;
    if (lo >= nch) return;
    const uint64_t hi = min(nch, lo + kCrcGroup);
    uint32_t s = 0;
    for (uint64_t c = lo; c < hi; ++c) s = gf2_apply(c == nch - 1 ? M_tail : M_chunk, s) ^ raw[c];
    group_raw[gidx] = s;
}

// CRC-32 of `size` bytes at device address `data` (16-byte aligned)
static uint32_t crc32_device(const uint8_t* data, uint64_t size, cudaStream_t& s, int num_sms) {
    static const std::vector<uint32_t> h_table = [] {
        std::vector<uint32_t> t(256);
        for (uint32_t i = 0; i < 256; ++i) t[i] = crc_table_entry(i);
        return t;
    }();
    if (size == 0) return 0;
    const uint64_t nch = (size + kCrcChunk - 1) / kCrcChunk;
    const uint64_t ngr = (nch + kCrcGroup - 1) / kCrcGroup;
    const uint64_t tail = size - (nch - 1) * kCrcChunk;  // bytes of the last chunk
    DevBuf table, raw, graw;
    table.ensure(256 * 4, s);
    raw.ensure(nch * 4, s);
    graw.ensure(ngr * 4, s);
    CK(cudaMemcpyAsync(table.p, h_table.data(), 1024, cudaMemcpyHostToDevice, s));
    k_crc_chunks<<<(unsigned)((nch + 255) / 256), 256, 0, s>>>(data, size, table.as<uint32_t>(), raw.as<uint32_t>());
    CKL("k_crc_chunks");
    const Gf2Mat M_chunk = crc_zeros_op(kCrcChunk), M_tail = crc_zeros_op(tail);
    k_crc_fold<<<(unsigned)((ngr + 127) / 128), 128, 0, s>>>(raw.as<uint32_t>(), nch, M_chunk, M_tail,
                                                           graw.as<uint32_t>());
    CKL("k_crc_fold");
    std::vector<uint32_t> h(ngr);
    CK(cudaMemcpyAsync(h.data(), graw.p, ngr * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    (void)num_sms;
    const Gf2Mat M_group = crc_zeros_op((uint64_t)kCrcGroup * kCrcChunk);
    const uint64_t last_len = size - (ngr - 1) * (uint64_t)kCrcGroup * kCrcChunk;
    const Gf2Mat M_last = crc_zeros_op(last_len);
    uint32_t st = 0;
    for (uint64_t j = 0; j < ngr; ++j) st = gf2_apply(j == ngr - 1 ? M_last : M_group, st) ^ h[j];
    return st ^ gf2_apply(crc_zeros_op(size), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
}

static void put_le(uint8_t* p, uint64_t v, int nbytes) {
    for (int i = 0; i < nbytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_le(const uint8_t* p, int nbytes) {
    uint64_t v = 0;
    for (int i = 0; i < nbytes; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

constexpr uint32_t kArtifactVersion = 1;  // persistence.hpp kArtifactFormatVersion
constexpr size_t kArtifactHeader = 44;

}  // namespace tpa

extern "C" {

int tpa_crc32(const void* data, uint64_t size, int flags, int device, uint32_t* out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output");
        if (size && !data) throw std::invalid_argument("null data");
        DeviceGuard dg(device);
        cudaStream_t s = nullptr;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct G {
            cudaStream_t s;
            ~G() {
                cudaStreamSynchronize(s);
                cudaStreamDestroy(s);
            }
        } sg{s};
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        DevBuf buf;
        const uint8_t* d = static_cast<const uint8_t*>(data);
        if (!(flags & TPA_DEVICE_PTRS) || (reinterpret_cast<uintptr_t>(data) & 15)) {
            buf.ensure(std::max<uint64_t>(size, 16), s);
            if (size)
                CK(cudaMemcpyAsync(buf.p, data, size, (flags & TPA_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice
                                                                               : cudaMemcpyHostToDevice, s));
            d = buf.as<uint8_t>();
        }
        *out = crc32_device(d, size, s, sms);
    });
}

int tpa_artifact_save(const tpa_artifact* a, const char* path) {
    return guard([&] {
        if (!a || !path) throw std::invalid_argument("null argument");
        if (!a->g) throw std::runtime_error("artifact outlived its graph handle");
        tpa_graph* g = a->g;
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        const uint64_t n = a->n;
        const uint64_t body = kArtifactHeader + 8 * n;
        // header + scores assembled in HBM (the CRC runs there), then one D2H into pinned memory
        uint8_t hdr[kArtifactHeader];
        std::memcpy(hdr, "TPA1", 4);
        put_le(hdr + 4, kArtifactVersion, 4);
        put_le(hdr + 8, n, 8);
        uint64_t bits;
        std::memcpy(&bits, &a->c, 8);
        put_le(hdr + 16, bits, 8);
        std::memcpy(&bits, &a->eps, 8);
        put_le(hdr + 24, bits, 8);
        put_le(hdr + 32, a->T, 4);
        put_le(hdr + 36, a->fingerprint, 8);
        DevBuf img;
        img.ensure(body + 16, g->stream);
        CK(cudaMemcpyAsync(img.p, hdr, kArtifactHeader, cudaMemcpyHostToDevice, g->stream));
        if (n)
            CK(cudaMemcpyAsync(img.as<uint8_t>() + kArtifactHeader, a->stranger.p, 8 * n, cudaMemcpyDeviceToDevice,
                               g->stream));
        const uint32_t crc = crc32_device(img.as<uint8_t>(), body, g->stream, g->num_sms);
        uint8_t* pinned = nullptr;
        CK(cudaMallocHost(&pinned, body + 4));
        struct Pin {
            uint8_t* p;
            ~Pin() { cudaFreeHost(p); }
        } pin{pinned};
        CK(cudaMemcpyAsync(pinned, img.p, body, cudaMemcpyDeviceToHost, g->stream));
        CK(cudaStreamSynchronize(g->stream));
        put_le(pinned + body, crc, 4);
        FILE* f = std::fopen(path, "wb");
        if (!f) throw std::runtime_error(std::string("cannot open for writing: ") + path);
        const size_t w = std::fwrite(pinned, 1, body + 4, f);
        const int ce = std::fclose(f);
        if (w != body + 4 || ce != 0) throw std::runtime_error(std::string("I/O error while writing ") + path);
    });
}

int tpa_artifact_load(tpa_graph* g, const char* path, tpa_artifact** out) {
    return guard([&] {
        if (!g || !path || !out) throw std::invalid_argument("null argument");
        require_whole(g, "tpa_artifact_load");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        FILE* f = std::fopen(path, "rb");
        if (!f) throw std::runtime_error(std::string("cannot open artifact: ") + path);
        struct Closer {
            FILE* f;
            ~Closer() { std::fclose(f); }
        } closer{f};
        std::fseek(f, 0, SEEK_END);
        const long len = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        if (len < 0) throw std::runtime_error(std::string("I/O error while reading ") + path);
        const uint64_t size = (uint64_t)len;
        uint8_t* pinned = nullptr;
        CK(cudaMallocHost(&pinned, std::max<uint64_t>(size, 1)));
        struct Pin {
            uint8_t* p;
            ~Pin() { cudaFreeHost(p); }
        } pin{pinned};
        if (size && std::fread(pinned, 1, size, f) != size)
            throw std::runtime_error(std::string("I/O error while reading ") + path);
        // persistence.cpp:103-117, in order
        if (size < 48) throw std::runtime_error(std::string("artifact truncated: ") + path);
        if (std::memcmp(pinned, "TPA1", 4) != 0) throw std::runtime_error(std::string("bad artifact magic: ") + path);
        const uint32_t version = (uint32_t)get_le(pinned + 4, 4);
        if (version != kArtifactVersion)
            throw std::runtime_error("unsupported artifact version " + std::to_string(version));
        const uint64_t n = get_le(pinned + 8, 8);
        // node ids are uint32 (graph.hpp NodeId); a larger count is corrupt and
        // would wrap 48 + 8n
        if (n > 0xffffffffull)
            throw std::runtime_error("artifact truncated or oversized: node count " + std::to_string(n) +
                                     " exceeds the uint32 node-id range");
        const uint64_t expected = 48 + 8 * n;
        if (size != expected)
            throw std::runtime_error("artifact truncated or oversized: expected " + std::to_string(expected) +
                                     " bytes, got " + std::to_string(size));
        DevBuf img;
        img.ensure(size + 16, g->stream);
        CK(cudaMemcpyAsync(img.p, pinned, size - 4, cudaMemcpyHostToDevice, g->stream));
        const uint32_t crc = crc32_device(img.as<uint8_t>(), size - 4, g->stream, g->num_sms);
        if ((uint32_t)get_le(pinned + size - 4, 4) != crc)
            throw std::runtime_error(std::string("artifact checksum mismatch: ") + path);
        auto art = std::make_unique<tpa_artifact>();
        art->g = g;
        art->n = n;
        uint64_t bits = get_le(pinned + 16, 8);
        std::memcpy(&art->c, &bits, 8);
        bits = get_le(pinned + 24, 8);
        std::memcpy(&art->eps, &bits, 8);
        art->T = (uint32_t)get_le(pinned + 32, 4);
        art->fingerprint = get_le(pinned + 36, 8);
        art->stranger.ensure(std::max<uint64_t>(8 * n, 8), g->stream);
        if (n)
            CK(cudaMemcpyAsync(art->stranger.p, img.as<uint8_t>() + kArtifactHeader, 8 * n, cudaMemcpyDeviceToDevice,
                               g->stream));
        CK(cudaStreamSynchronize(g->stream));
        g->artifacts.insert(art.get());
        *out = art.release();
    });
}

int tpa_artifact_info(const tpa_artifact* a, uint64_t* n, double* c, double* eps, uint32_t* T,
                      uint64_t* fingerprint) {
    return guard([&] {
        if (!a) throw std::invalid_argument("null artifact");
        if (n) *n = a->n;
        if (c) *c = a->c;
        if (eps) *eps = a->eps;
        if (T) *T = a->T;
        if (fingerprint) *fingerprint = a->fingerprint;
    });
}

int tpa_artifact_scores(const tpa_artifact* a, double* out, int flags) {
    return guard([&] {
        if (!a || !out) throw std::invalid_argument("null argument");
        if (!a->g) throw std::runtime_error("artifact outlived its graph handle");
        tpa_graph* g = a->g;
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        if (a->n)
            CK(cudaMemcpyAsync(out, a->stranger.p, 8 * a->n,
                               (flags & TPA_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                               g->stream));
        CK(cudaStreamSynchronize(g->stream));
    });
}

}  // extern "C"

// container.cpp — QGIR1 flat-binary circuit-set container (native parse/write).
//
// Reference: container.py:1-16 (format), write_binary container.py:71-84,
// read_binary container.py:87-115.  Layout, little-endian:
//   "QGIR1" | u32 capacity | u32 n_circ | u32 n_meta
//   | circ_type  int32 (n_circ, 3) | gate_type int32 (n_circ, capacity, 3)
//   | gate_param float64 (n_circ, capacity)
//   | n_meta x (u32 len, key UTF-8, u32 len, value UTF-8) in sorted key order
// The parser only validates and reports byte offsets, so the caller can map
// the file and hand the arrays to qg_plan_create without building Python
// objects per gate (1e8-record tensors).  Errors follow
// read_binary: bad magic, truncated file, trailing bytes -> ContainerFormatError.
#include <stdint.h>

#include <cstring>
#include <string>

#include "../../include/qgear_b200.h"

namespace {
thread_local std::string g_cerr;
int cfail(const std::string& m) {
    g_cerr = m;
    return QG_E_CONTAINER_FORMAT;
}
uint32_t rd32(const uint8_t* p) {
    uint32_t v;
    std::memcpy(&v, p, 4);  // the format is little-endian, as is every CUDA host
    return v;
}
constexpr char kMagic[] = "QGIR1";
constexpr int64_t kMagicLen = 5;
}  // namespace

extern "C" {

const char* qg_container_last_error(void) { return g_cerr.c_str(); }

int qg_qgir1_parse(const void* buf, int64_t len, qg_qgir1_info* out) {
    if (!buf || !out || len < 0) return cfail("NULL argument");
    const uint8_t* b = static_cast<const uint8_t*>(buf);
    if (len < kMagicLen || std::memcmp(b, kMagic, kMagicLen) != 0) return cfail("bad magic, not a QGIR1 file");
    int64_t off = kMagicLen;
    auto need = [&](int64_t n) { return n >= 0 && off + n <= len; };
    if (!need(12)) return cfail("truncated file");
    out->capacity = rd32(b + off);
    out->n_circ = rd32(b + off + 4);
    out->n_meta = rd32(b + off + 8);
    off += 12;
    const int64_t nc = out->n_circ, cap = out->capacity;
    out->headers_off = off;
    if (!need(nc * 12)) return cfail("truncated file");
    off += nc * 12;
    out->gate_type_off = off;
    if (!need(nc * cap * 12)) return cfail("truncated file");
    off += nc * cap * 12;
    out->gate_param_off = off;
    if (!need(nc * cap * 8)) return cfail("truncated file");
    off += nc * cap * 8;
    out->meta_off = off;
    for (uint32_t i = 0; i < out->n_meta; ++i)
        for (int kv = 0; kv < 2; ++kv) {
            if (!need(4)) return cfail("truncated file");
            const int64_t l = rd32(b + off);
            off += 4;
            if (!need(l)) return cfail("truncated file");
            off += l;
        }
    if (off != len) return cfail(std::to_string(len - off) + " trailing bytes");
    out->total_bytes = off;
    return QG_OK;
}

int64_t qg_qgir1_size(uint32_t capacity, uint32_t n_circ, uint32_t n_meta, const int64_t* meta_lens) {
    int64_t n = kMagicLen + 12 + (int64_t)n_circ * 12 + (int64_t)n_circ * capacity * 20;
    for (uint32_t i = 0; i < 2 * n_meta; ++i) n += 4 + (meta_lens ? meta_lens[i] : 0);
    return n;
}

int qg_qgir1_write(void* buf, int64_t len, uint32_t capacity, uint32_t n_circ, const int32_t* headers,
                   const int32_t* gate_type, const double* gate_param, uint32_t n_meta, const char* const* meta,
                   const int64_t* meta_lens) {
    if (!buf || (n_circ && (!headers || (capacity && (!gate_type || !gate_param)))) || (n_meta && (!meta || !meta_lens)))
        return cfail("NULL argument");
    if (len != qg_qgir1_size(capacity, n_circ, n_meta, meta_lens)) return cfail("buffer size mismatch");
    uint8_t* b = static_cast<uint8_t*>(buf);
    std::memcpy(b, kMagic, kMagicLen);
    int64_t off = kMagicLen;
    const uint32_t hdr[3] = {capacity, n_circ, n_meta};
    std::memcpy(b + off, hdr, 12);
    off += 12;
    std::memcpy(b + off, headers, (size_t)n_circ * 12);
    off += (int64_t)n_circ * 12;
    std::memcpy(b + off, gate_type, (size_t)n_circ * capacity * 12);
    off += (int64_t)n_circ * capacity * 12;
    std::memcpy(b + off, gate_param, (size_t)n_circ * capacity * 8);
    off += (int64_t)n_circ * capacity * 8;
    for (uint32_t i = 0; i < 2 * n_meta; ++i) {  // (key, value) pairs, caller sorts by key
        const uint32_t l = (uint32_t)meta_lens[i];
        std::memcpy(b + off, &l, 4);
        off += 4;
        std::memcpy(b + off, meta[i], l);
        off += l;
    }
    return QG_OK;
}

}  // extern "C"

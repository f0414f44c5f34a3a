// snapshot.cpp — SNKT tensor files and KV-cache snapshots,
// host C++ over the engine's own C-ABI.  Restates tensor.cpp:80-140 (the SNKT
// format: "SNKT" | u32 version=1 | u32 dtype=1 (f32) | u32 ndim | ndim x u64
// dims | row-major f32 payload, little-endian, tensor.hpp:86-91) and
// kv_cache.cpp:123-191 (manifest.json + k_l{l}_h{h}.snkt / v_l{l}_h{h}.snkt
// per slot, f32 [length][head_dim]).  Snapshots written here load in the
// reference and vice versa (tests/test_snapshot.py).  Replay reads each slot
// into pinned memory, uploads it once and converts it to bf16 on the device,
// pipelined across slots (host::append_slots_f32 in engine.cu).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "host_util.hpp"
#include "json_lite.hpp"

using sinkr::host::append_slots_f32;
using sinkr::host::fail;
using sinkr::host::guard;

namespace {

namespace fs = std::filesystem;

constexpr char kMagic[4] = {'S', 'N', 'K', 'T'};
constexpr uint32_t kVersion = 1, kDtypeF32 = 1, kMaxNdim = 64;

[[noreturn]] void bad_file(const std::string& path, const std::string& what) {
    fail(SINKR_RUNTIME_ERROR, "SNKT parse error in '" + path + "': " + what);
}

void check(sinkr_status st) {
    if (st != SINKR_OK) fail(st, sinkr_last_error());
}

uint64_t numel(const uint64_t* dims, size_t ndim) {
    uint64_t n = 1;
    for (size_t i = 0; i < ndim; ++i) {
        if (dims[i] != 0 && n > std::numeric_limits<uint64_t>::max() / dims[i])
            fail(SINKR_INVALID_ARGUMENT, "tensor element count overflows u64");
        n *= dims[i];
    }
    return n;
}

void write_snkt(const std::string& path, const uint64_t* dims, size_t ndim, const float* data) {
    if (ndim == 0) fail(SINKR_INVALID_ARGUMENT, "tensor needs at least one dimension");
    for (size_t i = 0; i < ndim; ++i)
        if (dims[i] == 0) fail(SINKR_INVALID_ARGUMENT, "tensor dimensions must be positive");
    const uint64_t n = numel(dims, ndim);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail(SINKR_RUNTIME_ERROR, "cannot open '" + path + "' for writing");
    const uint32_t hdr[3] = {kVersion, kDtypeF32, (uint32_t)ndim};
    out.write(kMagic, 4);
    out.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    out.write(reinterpret_cast<const char*>(dims), (std::streamsize)(8 * ndim));
    out.write(reinterpret_cast<const char*>(data), (std::streamsize)(n * 4));
    if (!out) fail(SINKR_RUNTIME_ERROR, "write failed for '" + path + "'");
}

// header only (data == nullptr) or header + payload into `data`
std::vector<uint64_t> read_snkt(const std::string& path, float* data, size_t capacity,
                                bool want_data) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(SINKR_RUNTIME_ERROR, "cannot open '" + path + "' for reading");
    char magic[4];
    in.read(magic, 4);
    if (in.gcount() != 4 || std::memcmp(magic, kMagic, 4) != 0) bad_file(path, "bad magic");
    auto u32 = [&](uint32_t& v) {
        in.read(reinterpret_cast<char*>(&v), 4);
        return in.gcount() == 4;
    };
    uint32_t version = 0, dtype = 0, ndim = 0;
    if (!u32(version)) bad_file(path, "truncated header (version)");
    if (version != kVersion) bad_file(path, "unsupported version " + std::to_string(version));
    if (!u32(dtype)) bad_file(path, "truncated header (dtype)");
    if (dtype != kDtypeF32) bad_file(path, "unsupported dtype " + std::to_string(dtype));
    if (!u32(ndim)) bad_file(path, "truncated header (ndim)");
    if (ndim == 0 || ndim > kMaxNdim) bad_file(path, "bad ndim " + std::to_string(ndim));
    std::vector<uint64_t> dims(ndim);
    for (uint32_t i = 0; i < ndim; ++i) {
        in.read(reinterpret_cast<char*>(&dims[i]), 8);
        if (in.gcount() != 8) bad_file(path, "truncated dims");
        if (dims[i] == 0) bad_file(path, "zero dim " + std::to_string(i));
    }
    if (!want_data) return dims;
    const uint64_t n = numel(dims.data(), dims.size());
    if (n > capacity) fail(SINKR_INVALID_ARGUMENT, "tensor larger than the destination buffer");
    in.read(reinterpret_cast<char*>(data), (std::streamsize)(n * 4));
    if ((uint64_t)in.gcount() != n * 4) bad_file(path, "short payload");
    if (in.peek() != std::ifstream::traits_type::eof()) bad_file(path, "trailing bytes");
    return dims;
}

std::string slot_file(const char* prefix, size_t layer, size_t head) {
    return std::string(prefix) + "_l" + std::to_string(layer) + "_h" + std::to_string(head) + ".snkt";
}

struct Manifest {
    sinkr_cache_config cfg{};
    size_t length = 0;
};

Manifest read_manifest(const fs::path& dir) {
    std::ifstream in(dir / "manifest.json", std::ios::binary);
    if (!in) fail(SINKR_RUNTIME_ERROR, "cannot open snapshot manifest in '" + dir.string() + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    sinkr::json::Value j;
    try {
        j = sinkr::json::parse(ss.str());
    } catch (const std::runtime_error& e) {
        fail(SINKR_RUNTIME_ERROR, std::string("snapshot manifest parse error: ") + e.what());
    }
    Manifest m;
    try {
        const auto& c = j.at("config");
        m.cfg.num_layers = c.at("num_layers").as_u64();
        m.cfg.num_q_heads = c.at("num_q_heads").as_u64();
        m.cfg.num_kv_heads = c.at("num_kv_heads").as_u64();
        m.cfg.head_dim = c.at("head_dim").as_u64();
        m.cfg.capacity = c.at("capacity").as_u64();
        m.cfg.num_seqs = 1;
        m.length = j.at("length").as_u64();
    } catch (const std::runtime_error& e) {
        fail(SINKR_RUNTIME_ERROR, std::string("snapshot manifest: ") + e.what());
    }
    return m;
}

void replay_into(sinkr_engine* e, size_t seq, const fs::path& dir, const Manifest& m) {
    sinkr_cache_config have{};
    check(sinkr_engine_config(e, &have));
    if (have.num_layers != m.cfg.num_layers || have.num_q_heads != m.cfg.num_q_heads ||
        have.num_kv_heads != m.cfg.num_kv_heads || have.head_dim != m.cfg.head_dim)
        fail(SINKR_INVALID_ARGUMENT, "snapshot shape does not match the engine");
    if (m.length > have.capacity)
        fail(SINKR_RUNTIME_ERROR, "kv cache overflow: slot at capacity " + std::to_string(have.capacity));
    const size_t D = m.cfg.head_dim, n = m.length * D;
    const std::vector<uint64_t> want = {m.length, D};
    // every slot's rows straight into the engine's pinned staging; the
    // upload and device conversion of slot i overlap the file reads of i+1
    append_slots_f32(e, seq, m.length, [&](size_t l, size_t h, float* k, float* v) {
        const auto kd = read_snkt((dir / slot_file("k", l, h)).string(), k, n, true);
        const auto vd = read_snkt((dir / slot_file("v", l, h)).string(), v, n, true);
        if (kd != want || vd != want)
            fail(SINKR_RUNTIME_ERROR, "snapshot tensor shape does not match manifest");
    });
}

}  // namespace

extern "C" {

uint64_t sinkr_snkt_file_size(const uint64_t* dims, size_t ndim) {
    uint64_t n = 1;
    for (size_t i = 0; i < ndim; ++i) n *= dims[i];
    return 4 + 4 + 4 + 4 + 8 * (uint64_t)ndim + 4 * n;
}

sinkr_status sinkr_write_tensor(const char* path, const uint64_t* dims, size_t ndim,
                                const float* data) {
    return guard([&] {
        if (!path || (ndim && !dims) || !data) fail(SINKR_INVALID_ARGUMENT, "null argument");
        write_snkt(path, dims, ndim, data);
    });
}

sinkr_status sinkr_read_tensor(const char* path, uint64_t* dims, size_t* ndim, float* data,
                               size_t capacity) {
    return guard([&] {
        if (!path || !dims || !ndim) fail(SINKR_INVALID_ARGUMENT, "null argument");
        const auto d = read_snkt(path, data, capacity, data != nullptr);
        for (size_t i = 0; i < d.size(); ++i) dims[i] = d[i];
        *ndim = d.size();
    });
}

sinkr_status sinkr_save_snapshot(sinkr_engine* e, size_t seq, const char* dir_c) {
    return guard([&] {
        if (!e || !dir_c) fail(SINKR_INVALID_ARGUMENT, "null argument");
        const fs::path dir(dir_c);
        sinkr_cache_config c{};
        check(sinkr_engine_config(e, &c));
        size_t len = 0;
        check(sinkr_kv_token_count(e, seq, &len));  // ragged slots throw, as token_count() does
        fs::create_directories(dir);
        const size_t D = c.head_dim;
        std::vector<float> k(len * D), v(len * D);
        for (size_t l = 0; l < c.num_layers; ++l) {
            for (size_t h = 0; h < c.num_kv_heads; ++h) {
                if (len) check(sinkr_kv_read(e, seq, l, h, 0, len, k.data(), v.data()));
                const uint64_t dims[2] = {len, D};
                if (len == 0) fail(SINKR_INVALID_ARGUMENT, "tensor dimensions must be positive");
                write_snkt((dir / slot_file("k", l, h)).string(), dims, 2, k.data());
                write_snkt((dir / slot_file("v", l, h)).string(), dims, 2, v.data());
            }
        }
        using sinkr::json::num;
        std::string j = "{\n  \"version\": 1,\n  \"config\": {\n";
        j += "    \"num_layers\": " + num((unsigned long long)c.num_layers) + ",\n";
        j += "    \"num_q_heads\": " + num((unsigned long long)c.num_q_heads) + ",\n";
        j += "    \"num_kv_heads\": " + num((unsigned long long)c.num_kv_heads) + ",\n";
        j += "    \"head_dim\": " + num((unsigned long long)c.head_dim) + ",\n";
        j += "    \"capacity\": " + num((unsigned long long)c.capacity) + "\n  },\n";
        j += "  \"length\": " + num((unsigned long long)len) + "\n}\n";
        std::ofstream out(dir / "manifest.json", std::ios::binary | std::ios::trunc);
        if (!out) fail(SINKR_RUNTIME_ERROR, "cannot write snapshot manifest");
        out << j;
        if (!out) fail(SINKR_RUNTIME_ERROR, "cannot write snapshot manifest");
    });
}

sinkr_status sinkr_load_snapshot(const char* dir_c, int device, sinkr_engine** out) {
    return guard([&] {
        if (!dir_c || !out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        const fs::path dir(dir_c);
        const Manifest m = read_manifest(dir);
        sinkr_engine* e = nullptr;
        check(sinkr_engine_create(&m.cfg, device, &e));
        try {
            replay_into(e, 0, dir, m);
        } catch (...) {
            sinkr_engine_destroy(e);
            throw;
        }
        *out = e;
    });
}

sinkr_status sinkr_load_snapshot_into(sinkr_engine* e, size_t seq, const char* dir_c) {
    return guard([&] {
        if (!e || !dir_c) fail(SINKR_INVALID_ARGUMENT, "null argument");
        const fs::path dir(dir_c);
        replay_into(e, seq, dir, read_manifest(dir));
    });
}

}  // extern "C"

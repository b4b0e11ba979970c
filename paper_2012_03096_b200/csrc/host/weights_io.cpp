// weights_io.cpp -- PBKD weight container (format: include/pbkd/weights_io.hpp;
// reference: proj/src/weights_io.cpp:68-319).  Host-side only: the GPU engine
// exchanges weights with callers as flat arrays in for_each_array order; this
// file converts networks to and from the reference's on-disk checkpoints.
#include "pbkd/weights_io.hpp"

#include <cstring>
#include <fstream>
#include <iterator>
#include <map>
#include <set>

#include "pbkd/replacement.hpp"
#include "pbkd/tensor.hpp"

namespace pbkd {

namespace {

constexpr char kMagic[4] = {'P', 'B', 'K', 'D'};
constexpr uint32_t kVersion = 1;

template <class T>
void put_le(std::string& out, T v) {
    for (size_t i = 0; i < sizeof(T); ++i) out.push_back(static_cast<char>((static_cast<uint64_t>(v) >> (8 * i)) & 0xff));
}

// bounds-checked little-endian cursor over the file bytes
class Cursor {
public:
    Cursor(const std::string& bytes, const std::string& origin) : b_(bytes), origin_(origin) {}
    template <class T>
    T get(const char* what) {
        need(sizeof(T), what);
        uint64_t v = 0;
        for (size_t i = 0; i < sizeof(T); ++i) v |= static_cast<uint64_t>(static_cast<unsigned char>(b_[at_ + i])) << (8 * i);
        at_ += sizeof(T);
        return static_cast<T>(v);
    }
    const char* take(size_t n, const char* what) {
        need(n, what);
        const char* p = b_.data() + at_;
        at_ += n;
        return p;
    }
    size_t left() const { return b_.size() - at_; }

private:
    void need(size_t n, const char* what) const {
        if (b_.size() - at_ < n) throw WeightsError(origin_ + ": truncated file while reading " + what);
    }
    const std::string& b_;
    std::string origin_;
    size_t at_ = 0;
};

std::string read_file(const std::string& path, const char* why) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw WeightsError(path + ": cannot open" + why);
    return std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

size_t volume(const std::vector<uint32_t>& dims) {
    size_t v = 1;
    for (uint32_t d : dims) v *= d;
    return v;
}

// name -> dims of every array a block stores
std::map<std::string, std::vector<uint32_t>> block_signature(Block& b) {
    std::map<std::string, std::vector<uint32_t>> sig;
    for_each_block_array(b, [&](const std::string& name, Tensor& t) {
        sig[name] = {static_cast<uint32_t>(t.n), static_cast<uint32_t>(t.c), static_cast<uint32_t>(t.h),
                     static_cast<uint32_t>(t.w)};
    });
    return sig;
}

}  // namespace

void save_weights(const std::string& path, const std::vector<NamedArray>& arrays) {
    std::string out(kMagic, 4);
    put_le<uint32_t>(out, kVersion);
    put_le<uint32_t>(out, static_cast<uint32_t>(arrays.size()));
    for (const NamedArray& a : arrays) {
        if (a.name.size() > 0xffff) throw WeightsError(path + ": array name too long: " + a.name.substr(0, 64));
        if (a.dims.empty()) throw WeightsError(path + ": array '" + a.name + "' has no dims");
        for (uint32_t d : a.dims)
            if (d == 0) throw WeightsError(path + ": array '" + a.name + "' has a zero dim");
        if (volume(a.dims) != a.data.size())
            throw WeightsError(path + ": array '" + a.name + "' dims do not match payload size");
        put_le<uint16_t>(out, static_cast<uint16_t>(a.name.size()));
        out += a.name;
        out.push_back(static_cast<char>(a.dims.size()));
        for (uint32_t d : a.dims) put_le<uint32_t>(out, d);
        const size_t at = out.size();
        out.resize(at + 4 * a.data.size());
        std::memcpy(&out[at], a.data.data(), 4 * a.data.size());  // little-endian host
    }
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw WeightsError(path + ": cannot open for writing");
    f.write(out.data(), static_cast<std::streamsize>(out.size()));
    if (!f) throw WeightsError(path + ": write failed");
}

std::vector<NamedArray> load_weights(const std::string& path) {
    const std::string bytes = read_file(path, "");
    Cursor c(bytes, path);
    if (std::memcmp(c.take(4, "magic"), kMagic, 4) != 0) throw WeightsError(path + ": not a weights file (bad magic)");
    const uint32_t version = c.get<uint32_t>("version");
    if (version != kVersion) throw WeightsError(path + ": unsupported format version " + std::to_string(version));
    const uint32_t count = c.get<uint32_t>("array count");
    std::vector<NamedArray> arrays;
    arrays.reserve(count);
    for (uint32_t i = 0; i < count; ++i) {
        NamedArray a;
        const uint16_t len = c.get<uint16_t>("name length");
        a.name.assign(c.take(len, "array name"), len);
        const uint8_t rank = c.get<uint8_t>("rank");
        if (rank == 0 || rank > 8)
            throw WeightsError(path + ": array '" + a.name + "' has implausible rank " + std::to_string(rank));
        for (uint8_t d = 0; d < rank; ++d) {
            a.dims.push_back(c.get<uint32_t>("dims"));
            if (a.dims.back() == 0) throw WeightsError(path + ": array '" + a.name + "' has a zero dim");
        }
        const size_t n = volume(a.dims);
        a.data.resize(n);
        std::memcpy(a.data.data(), c.take(4 * n, "payload"), 4 * n);
        arrays.push_back(std::move(a));
    }
    if (c.left() != 0) throw WeightsError(path + ": " + std::to_string(c.left()) + " trailing bytes after the last array");
    return arrays;
}

std::vector<NamedArray> arrays_from_network(const Network& net) {
    std::vector<NamedArray> out;
    for_each_array(const_cast<Network&>(net), [&](const std::string& name, Tensor& t) {
        out.push_back(NamedArray{name,
                                 {static_cast<uint32_t>(t.n), static_cast<uint32_t>(t.c), static_cast<uint32_t>(t.h),
                                  static_cast<uint32_t>(t.w)},
                                 t.data});
    });
    return out;
}

void load_into_network(Network& net, const std::vector<NamedArray>& arrays, const std::string& origin) {
    std::map<std::string, const NamedArray*> by_name;
    for (const NamedArray& a : arrays)
        if (!by_name.emplace(a.name, &a).second) throw WeightsError(origin + ": duplicate array '" + a.name + "'");
    // validate everything first, then assign
    std::vector<std::pair<Tensor*, const NamedArray*>> todo;
    for_each_array(net, [&](const std::string& name, Tensor& t) {
        const auto it = by_name.find(name);
        if (it == by_name.end())
            throw WeightsError(origin + ": missing array '" + name + "' required by network '" + net.name + "'");
        const NamedArray& a = *it->second;
        const bool ok = a.dims.size() == 4 && a.dims[0] == static_cast<uint32_t>(t.n) &&
                        a.dims[1] == static_cast<uint32_t>(t.c) && a.dims[2] == static_cast<uint32_t>(t.h) &&
                        a.dims[3] == static_cast<uint32_t>(t.w) && volume(a.dims) == t.data.size();
        if (!ok) throw WeightsError(origin + ": array '" + name + "' has the wrong shape for tensor " + t.shape_str());
        todo.emplace_back(&t, &a);
    });
    if (todo.size() != arrays.size())
        for (const NamedArray& a : arrays) {
            bool used = false;
            for (const auto& p : todo) used = used || p.second == &a;
            if (!used) throw WeightsError(origin + ": array '" + a.name + "' does not belong to network '" + net.name + "'");
        }
    for (auto& p : todo) p.first->data = p.second->data;
}

Network rebuild_network_from_arrays(const Network& teacher_structure, const std::vector<NamedArray>& arrays,
                                    const std::string& origin) {
    std::map<std::string, std::map<std::string, std::vector<uint32_t>>> by_block;  // block -> name -> dims
    for (const NamedArray& a : arrays) {
        const size_t slash = a.name.find('/');
        if (slash == std::string::npos || slash == 0)
            throw WeightsError(origin + ": array name '" + a.name + "' has no block prefix");
        by_block[a.name.substr(0, slash)][a.name] = a.dims;
    }
    Network out = teacher_structure;
    for (Block& b : out.blocks) {
        const auto it = by_block.find(b.name);
        if (it == by_block.end()) throw WeightsError(origin + ": no arrays for block '" + b.name + "'");
        if (block_signature(b) == it->second) continue;  // teacher-structured block
        // a replacement block: the candidate whose stored arrays (names under
        // this block's name, shapes) are exactly the file's
        bool found = false;
        for (CandidateKind kind : {CandidateKind::TwoLayer, CandidateKind::ThreeLayer, CandidateKind::TwoLayerSkip,
                                   CandidateKind::ThreeLayerSkip}) {
            Block cand = build_candidate(kind, b.in_channels, b.out_channels, b.stride, 0).block;
            cand.name = b.name;
            if (block_signature(cand) != it->second) continue;
            cand.replaceable = false;
            b = std::move(cand);
            found = true;
            break;
        }
        if (!found)
            throw WeightsError(origin + ": block '" + b.name +
                               "' matches neither the teacher structure nor a replacement candidate");
    }
    load_into_network(out, arrays, origin);
    return out;
}

uint64_t file_hash(const std::string& path) {
    const std::string bytes = read_file(path, " for hashing");
    return fnv1a64(bytes.data(), bytes.size());
}

}  // namespace pbkd

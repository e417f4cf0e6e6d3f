// keyfile.hpp -- the reference CLI's key-file formats, restated for the B200
// command line tool (format: proj/include/comerge/io.hpp:11-20; reader and
// writer behaviour: proj/src/io.cpp:33-133).
//
//   text    one unsigned decimal integer per line ('\n', optional '\r'),
//           blank lines tolerated
//   binary  "CRMG" | version u8 = 1 | flags u8 | count u64 LE | count x u64 LE
//
// The format is detected from the magic bytes.  Malformed or unreadable
// files throw keyfile_error (CLI exit 3); unsorted keys throw
// std::invalid_argument when validation is on (CLI exit 2).
#pragma once

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

namespace comerge_cli {

struct keyfile_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class key_format { text, binary };

struct keys_file {
    std::vector<std::uint64_t> keys;
    key_format format = key_format::text;
};

inline constexpr char kMagic[4] = {'C', 'R', 'M', 'G'};
inline constexpr unsigned char kVersion = 1;
inline constexpr std::size_t kHeader = 4 + 1 + 1 + 8;

inline std::uint64_t load_le64(const unsigned char* p) {
    std::uint64_t x = 0;
    for (int i = 7; i >= 0; --i) x = (x << 8) | p[i];
    return x;
}

inline void store_le64(std::uint64_t x, unsigned char* p) {
    for (int i = 0; i < 8; ++i, x >>= 8) p[i] = static_cast<unsigned char>(x & 0xffu);
}

inline keys_file read_keys(const std::string& path, bool validate) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw keyfile_error(path + ": cannot open for reading");
    const std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (in.bad()) throw keyfile_error(path + ": read failed");
    keys_file f;
    if (data.size() >= 4 && std::memcmp(data.data(), kMagic, 4) == 0) {
        f.format = key_format::binary;
        if (data.size() < kHeader) throw keyfile_error(path + ": truncated header");
        const auto* u = reinterpret_cast<const unsigned char*>(data.data());
        if (u[4] != kVersion)
            throw keyfile_error(path + ": unsupported format version " + std::to_string(u[4]));
        const std::uint64_t count = load_le64(u + 6);
        const std::uint64_t body = data.size() - kHeader;
        if (body % 8 != 0 || body / 8 != count)
            throw keyfile_error(path + ": declared key count does not match payload length");
        f.keys.resize(count);
        for (std::uint64_t t = 0; t < count; ++t) f.keys[t] = load_le64(u + kHeader + 8 * t);
    } else {
        std::size_t pos = 0, line = 0;
        while (pos < data.size()) {
            std::size_t eol = data.find('\n', pos);
            if (eol == std::string::npos) eol = data.size();
            ++line;
            std::size_t end = eol;
            if (end > pos && data[end - 1] == '\r') --end;
            if (end > pos) {
                std::uint64_t v = 0;
                const auto [stop, ec] = std::from_chars(data.data() + pos, data.data() + end, v);
                if (ec != std::errc{} || stop != data.data() + end)
                    throw keyfile_error(path + ":" + std::to_string(line) +
                                        ": expected one unsigned decimal integer per line");
                f.keys.push_back(v);
            }
            pos = eol + 1;
        }
    }
    if (validate && !std::is_sorted(f.keys.begin(), f.keys.end()))
        throw std::invalid_argument(path + ": keys are not nondecreasing");
    return f;
}

inline void write_keys(const std::string& path, const std::vector<std::uint64_t>& keys,
                       key_format format) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw keyfile_error(path + ": cannot open for writing");
    std::string buf;
    if (format == key_format::binary) {
        buf.resize(kHeader + 8 * keys.size());
        auto* u = reinterpret_cast<unsigned char*>(buf.data());
        std::memcpy(u, kMagic, 4);
        u[4] = kVersion;
        u[5] = 0;  // flags
        store_le64(keys.size(), u + 6);
        for (std::size_t t = 0; t < keys.size(); ++t) store_le64(keys[t], u + kHeader + 8 * t);
    } else {
        buf.reserve(keys.size() * 8);
        char digits[24];
        for (const std::uint64_t k : keys) {
            const auto [end, ec] = std::to_chars(digits, digits + sizeof(digits), k);
            buf.append(digits, end);
            buf.push_back('\n');
        }
    }
    out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
    out.flush();
    if (!out) throw keyfile_error(path + ": write failed");
}

}  // namespace comerge_cli

// Safetensors-layout container, as LAYOUT ONLY: the header, the entry table
// and payload byte ranges. Payload bytes never pass through host containers
// on the B200 path — they live in device (or pinned host) buffers and are
// moved by the gather kernel. Byte format = R/src/container.cpp:62-100:
//   u64 LE header length | compact JSON header (sorted keys, "__metadata__"
//   optional) space-padded so (8 + len) % 8 == 0 | payload, tensors packed in
//   lexicographic name order.
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <string>
#include <vector>

namespace tailor {

enum class Dtype : int { BF16 = 0, F32 = 1 };
std::size_t dtype_size(Dtype d);
const char* dtype_name(Dtype d);

struct EntryDecl {
    std::string name;
    Dtype dtype = Dtype::F32;
    std::vector<std::int64_t> shape;
    std::int64_t numel() const {
        std::int64_t n = 1;
        for (auto d : shape) n *= d;
        return n;
    }
};

struct Entry {
    std::string name;
    Dtype dtype = Dtype::F32;
    std::vector<std::int64_t> shape;
    std::uint64_t begin = 0; // payload-relative
    std::uint64_t end = 0;
    std::uint64_t bytes() const { return end - begin; }
};

struct ContainerLayout {
    std::map<std::string, std::string> metadata;
    std::vector<Entry> entries; // lexicographic by name
    std::string header;         // padded JSON, exactly as written
    std::uint64_t payload_bytes = 0;

    std::uint64_t payload_offset() const { return 8 + header.size(); }
    std::uint64_t file_bytes() const { return payload_offset() + payload_bytes; }
    const Entry* find(const std::string& name) const;
    // The 8-byte length prefix followed by the padded header.
    std::string prefix() const;
};

// Builds the layout a writer would produce for these declarations.
ContainerLayout layout_for(std::vector<EntryDecl> decls, std::map<std::string, std::string> metadata = {});

// Reads and validates only the header of a container file (never the
// payload): ranges ascend in name order, tile the payload exactly and match
// each entry's shape (R/src/container.cpp:102-159 checks, minus the copy).
ContainerLayout read_layout(const std::filesystem::path& path);
ContainerLayout parse_layout(const std::string& prefix_and_header, std::uint64_t file_size, const std::string& origin);

} // namespace tailor

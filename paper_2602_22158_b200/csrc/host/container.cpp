// Container layout: header rendering and validation (see tailor/container.hpp).
#include "tailor/container.hpp"

#include <algorithm>
#include <cstdio>
#include <fstream>

#include <json.hpp>

#include "tailor/errors.hpp"

namespace tailor {

using nlohmann::json;

std::size_t dtype_size(Dtype d) { return d == Dtype::BF16 ? 2u : 4u; }
const char* dtype_name(Dtype d) { return d == Dtype::BF16 ? "BF16" : "F32"; }

namespace {

Dtype dtype_from(const std::string& s, const std::string& origin) {
    if (s == "BF16") return Dtype::BF16;
    if (s == "F32") return Dtype::F32;
    fail(ErrorKind::CorruptContainer, origin + ": unsupported dtype '" + s + "'");
}

std::string render_header(const ContainerLayout& c) {
    // nlohmann's object is a std::map: keys come out sorted, matching the
    // reference writer byte for byte (same library, same dump()).
    json h = json::object();
    if (!c.metadata.empty()) {
        json meta = json::object();
        for (const auto& [k, v] : c.metadata) meta[k] = v;
        h["__metadata__"] = std::move(meta);
    }
    for (const auto& e : c.entries) {
        json offs = json::array({static_cast<std::int64_t>(e.begin), static_cast<std::int64_t>(e.end)});
        h[e.name] = json{{"dtype", dtype_name(e.dtype)}, {"shape", e.shape}, {"data_offsets", std::move(offs)}};
    }
    std::string s = h.dump();
    s.append((8 - (8 + s.size()) % 8) % 8, ' ');
    return s;
}

} // namespace

const Entry* ContainerLayout::find(const std::string& name) const {
    auto it = std::lower_bound(entries.begin(), entries.end(), name,
                               [](const Entry& e, const std::string& n) { return e.name < n; });
    return (it != entries.end() && it->name == name) ? &*it : nullptr;
}

std::string ContainerLayout::prefix() const {
    std::string out(8, '\0');
    const std::uint64_t n = header.size();
    for (int i = 0; i < 8; ++i) out[static_cast<std::size_t>(i)] = static_cast<char>((n >> (8 * i)) & 0xFF);
    return out + header;
}

ContainerLayout layout_for(std::vector<EntryDecl> decls, std::map<std::string, std::string> metadata) {
    std::sort(decls.begin(), decls.end(), [](const EntryDecl& a, const EntryDecl& b) { return a.name < b.name; });
    ContainerLayout c;
    c.metadata = std::move(metadata);
    std::uint64_t off = 0;
    for (std::size_t i = 0; i < decls.size(); ++i) {
        if (i > 0 && decls[i].name == decls[i - 1].name)
            fail(ErrorKind::Geometry, "duplicate tensor name in container");
        const std::uint64_t n = static_cast<std::uint64_t>(decls[i].numel()) * dtype_size(decls[i].dtype);
        c.entries.push_back({decls[i].name, decls[i].dtype, decls[i].shape, off, off + n});
        off += n;
    }
    c.payload_bytes = off;
    c.header = render_header(c);
    return c;
}

ContainerLayout parse_layout(const std::string& buf, std::uint64_t file_size, const std::string& origin) {
    const auto corrupt = [&](const std::string& what) { fail(ErrorKind::CorruptContainer, origin + ": " + what); };
    if (buf.size() < 8 || file_size < 8) corrupt("shorter than the 8-byte header length");
    std::uint64_t hlen = 0;
    for (int i = 0; i < 8; ++i) hlen |= static_cast<std::uint64_t>(static_cast<unsigned char>(buf[static_cast<std::size_t>(i)])) << (8 * i);
    if (hlen > file_size - 8) corrupt("header length exceeds file size");
    if (buf.size() < 8 + hlen) corrupt("truncated header");
    json h;
    try {
        h = json::parse(buf.begin() + 8, buf.begin() + 8 + static_cast<std::ptrdiff_t>(hlen));
    } catch (const json::exception& e) {
        corrupt(std::string("header is not valid JSON (") + e.what() + ")");
    }
    if (!h.is_object()) corrupt("header is not a JSON object");
    ContainerLayout c;
    c.header = buf.substr(8, hlen);
    const std::uint64_t payload = file_size - 8 - hlen;
    std::uint64_t expect = 0;
    for (const auto& [name, info] : h.items()) {
        if (name == "__metadata__") {
            if (!info.is_object()) corrupt("__metadata__ is not an object");
            for (const auto& [k, v] : info.items()) {
                if (!v.is_string()) corrupt("__metadata__ values must be strings");
                c.metadata[k] = v.get<std::string>();
            }
            continue;
        }
        if (!info.is_object() || !info.contains("dtype") || !info.contains("shape") || !info.contains("data_offsets"))
            corrupt("tensor '" + name + "' entry is malformed");
        Entry e;
        e.name = name;
        try {
            e.dtype = dtype_from(info["dtype"].get<std::string>(), origin);
            e.shape = info["shape"].get<std::vector<std::int64_t>>();
            const auto o = info["data_offsets"].get<std::vector<std::int64_t>>();
            if (o.size() != 2 || o[0] < 0 || o[0] > o[1]) corrupt("tensor '" + name + "' has invalid offsets");
            e.begin = static_cast<std::uint64_t>(o[0]);
            e.end = static_cast<std::uint64_t>(o[1]);
        } catch (const json::exception& ex) {
            corrupt("tensor '" + name + "' entry is malformed (" + ex.what() + ")");
        }
        if (e.begin != expect) corrupt("tensor '" + name + "' does not start where the previous range ended");
        if (e.end > payload) corrupt("tensor '" + name + "' extends past the payload");
        std::int64_t numel = 1;
        for (auto d : e.shape) numel *= d;
        if (e.bytes() != static_cast<std::uint64_t>(numel) * dtype_size(e.dtype))
            corrupt("tensor '" + name + "' byte range does not match its shape");
        expect = e.end;
        c.entries.push_back(std::move(e));
    }
    if (expect != payload) corrupt("payload size does not match the declared ranges");
    c.payload_bytes = payload;
    return c;
}

ContainerLayout read_layout(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(ErrorKind::MissingArtifact, "cannot open '" + path.string() + "'");
    std::error_code ec;
    const std::uint64_t size = std::filesystem::file_size(path, ec);
    if (ec) fail(ErrorKind::Storage, "cannot stat '" + path.string() + "'");
    std::string buf(8, '\0');
    in.read(buf.data(), 8);
    if (in.gcount() != 8) fail(ErrorKind::CorruptContainer, path.string() + ": shorter than the 8-byte header length");
    std::uint64_t hlen = 0;
    for (int i = 0; i < 8; ++i) hlen |= static_cast<std::uint64_t>(static_cast<unsigned char>(buf[static_cast<std::size_t>(i)])) << (8 * i);
    if (hlen > size - 8) fail(ErrorKind::CorruptContainer, path.string() + ": header length exceeds file size");
    buf.resize(8 + hlen);
    in.read(buf.data() + 8, static_cast<std::streamsize>(hlen));
    if (static_cast<std::uint64_t>(in.gcount()) != hlen) fail(ErrorKind::Storage, "read failed for '" + path.string() + "'");
    return parse_layout(buf, size, path.string());
}

} // namespace tailor

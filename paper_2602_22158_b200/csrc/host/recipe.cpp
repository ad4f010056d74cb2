// Strict YAML merge-recipe schema (R/src/recipe.cpp:67-169). yaml-cpp is not
// in this image, so this file carries a small YAML reader for the subset the
// schema uses — block maps and sequences, flow [..] / {..}, plain and quoted
// scalars, comments — and an emitter in yaml-cpp's block style. Schema
// errors name the offending field, as the reference's do.
#include <cctype>
#include <set>

#include "tailor/errors.hpp"
#include "tailor/merge.hpp"

namespace tailor {

namespace {

struct Node {
    enum Kind { Null, Scalar, Seq, Map } kind = Null;
    std::string text;
    bool quoted = false;
    std::vector<Node> items;
    std::vector<std::pair<std::string, Node>> fields;
    const Node* get(const std::string& k) const {
        for (const auto& [key, v] : fields)
            if (key == k) return &v;
        return nullptr;
    }
};

[[noreturn]] void yaml_error(const std::string& what) { fail(ErrorKind::Recipe, "invalid YAML: " + what); }

struct Line {
    int indent;
    std::string text; // comment-stripped, right-trimmed
    int number;
};

std::string strip_comment(const std::string& s) {
    char quote = 0;
    for (std::size_t i = 0; i < s.size(); ++i) {
        const char c = s[i];
        if (quote) {
            if (c == quote) quote = 0;
            continue;
        }
        if (c == '"' || c == '\'') quote = c;
        else if (c == '#' && (i == 0 || s[i - 1] == ' ' || s[i - 1] == '\t')) return s.substr(0, i);
    }
    return s;
}

std::string rtrim(std::string s) {
    while (!s.empty() && std::isspace(static_cast<unsigned char>(s.back()))) s.pop_back();
    return s;
}

std::string trim(const std::string& s) {
    std::size_t b = 0;
    while (b < s.size() && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
    return rtrim(s.substr(b));
}

// ---- flow / scalar parsing ----
class Flow {
  public:
    explicit Flow(const std::string& s) : s_(s) {}
    Node parse_all() {
        Node n = value(false);
        ws();
        if (i_ != s_.size()) yaml_error("unexpected trailing text '" + s_.substr(i_) + "'");
        return n;
    }

  private:
    void ws() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t')) ++i_;
    }
    Node value(bool in_flow) {
        ws();
        if (i_ >= s_.size()) return Node{};
        if (s_[i_] == '[') return seq();
        if (s_[i_] == '{') return map();
        return scalar(in_flow, false);
    }
    Node scalar(bool in_flow, bool is_key) {
        ws();
        Node n;
        n.kind = Node::Scalar;
        if (i_ < s_.size() && (s_[i_] == '"' || s_[i_] == '\'')) {
            const char q = s_[i_++];
            n.quoted = true;
            while (true) {
                if (i_ >= s_.size()) yaml_error("unterminated quoted scalar");
                const char c = s_[i_++];
                if (c == q) {
                    if (q == '\'' && i_ < s_.size() && s_[i_] == '\'') {
                        n.text.push_back('\'');
                        ++i_;
                        continue;
                    }
                    break;
                }
                if (q == '"' && c == '\\') {
                    if (i_ >= s_.size()) yaml_error("bad escape");
                    const char e = s_[i_++];
                    n.text.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e);
                    continue;
                }
                n.text.push_back(c);
            }
            return n;
        }
        const std::size_t b = i_;
        while (i_ < s_.size()) {
            const char c = s_[i_];
            if (in_flow && (c == ',' || c == ']' || c == '}')) break;
            if (is_key && c == ':' && (i_ + 1 == s_.size() || s_[i_ + 1] == ' ')) break;
            ++i_;
        }
        n.text = trim(s_.substr(b, i_ - b));
        if (n.text.empty() || n.text == "~" || n.text == "null") {
            n.kind = Node::Null;
            n.text.clear();
        }
        return n;
    }
    Node seq() {
        Node n;
        n.kind = Node::Seq;
        ++i_;
        ws();
        if (i_ < s_.size() && s_[i_] == ']') {
            ++i_;
            return n;
        }
        while (true) {
            n.items.push_back(value(true));
            ws();
            if (i_ >= s_.size()) yaml_error("unterminated flow sequence");
            if (s_[i_] == ',') {
                ++i_;
                continue;
            }
            if (s_[i_] == ']') {
                ++i_;
                return n;
            }
            yaml_error("expected ',' or ']' in flow sequence");
        }
    }
    Node map() {
        Node n;
        n.kind = Node::Map;
        ++i_;
        ws();
        if (i_ < s_.size() && s_[i_] == '}') {
            ++i_;
            return n;
        }
        while (true) {
            Node k = scalar(true, true);
            ws();
            if (i_ >= s_.size() || s_[i_] != ':') yaml_error("expected ':' in flow mapping");
            ++i_;
            for (const auto& f : n.fields)
                if (f.first == k.text) yaml_error("duplicate key '" + k.text + "'");
            n.fields.emplace_back(k.text, value(true));
            ws();
            if (i_ >= s_.size()) yaml_error("unterminated flow mapping");
            if (s_[i_] == ',') {
                ++i_;
                continue;
            }
            if (s_[i_] == '}') {
                ++i_;
                return n;
            }
            yaml_error("expected ',' or '}' in flow mapping");
        }
    }
    const std::string& s_;
    std::size_t i_ = 0;
};

// Splits "key: rest" at the first ': ' (or trailing ':') outside quotes and
// flow brackets. Returns false if the line is not a mapping entry.
bool split_key(const std::string& t, std::string& key, std::string& rest) {
    char quote = 0;
    int depth = 0;
    for (std::size_t i = 0; i < t.size(); ++i) {
        const char c = t[i];
        if (quote) {
            if (c == quote) quote = 0;
            continue;
        }
        if (c == '"' || c == '\'') quote = c;
        else if (c == '[' || c == '{') ++depth;
        else if (c == ']' || c == '}') --depth;
        else if (c == ':' && depth == 0 && (i + 1 == t.size() || t[i + 1] == ' ')) {
            std::string k = trim(t.substr(0, i));
            if (k.size() >= 2 && (k.front() == '"' || k.front() == '\'') && k.back() == k.front()) k = k.substr(1, k.size() - 2);
            key = k;
            rest = trim(t.substr(i + 1));
            return !key.empty();
        }
    }
    return false;
}

class Block {
  public:
    explicit Block(std::vector<Line> lines) : lines_(std::move(lines)) {}
    Node parse() {
        if (lines_.empty()) return Node{};
        Node n = node_at(lines_[0].indent);
        if (pos_ != lines_.size()) yaml_error("unexpected content at line " + std::to_string(lines_[pos_].number));
        return n;
    }

  private:
    bool is_item(const Line& l) const { return l.text == "-" || l.text.rfind("- ", 0) == 0; }

    Node node_at(int indent) {
        const Line& l = lines_[pos_];
        if (l.indent != indent) yaml_error("bad indentation at line " + std::to_string(l.number));
        if (is_item(l)) return seq_at(indent);
        std::string k, r;
        if (split_key(l.text, k, r)) return map_at(indent);
        ++pos_;
        return Flow(l.text).parse_all();
    }

    Node value_after(const std::string& rest, int indent, bool allow_same_indent_seq) {
        if (!rest.empty()) return Flow(rest).parse_all();
        if (pos_ < lines_.size()) {
            const Line& nx = lines_[pos_];
            if (nx.indent > indent) return node_at(nx.indent);
            if (allow_same_indent_seq && nx.indent == indent && is_item(nx)) return seq_at(indent);
        }
        return Node{};
    }

    Node map_at(int indent) {
        Node n;
        n.kind = Node::Map;
        while (pos_ < lines_.size() && lines_[pos_].indent == indent && !is_item(lines_[pos_])) {
            std::string k, r;
            if (!split_key(lines_[pos_].text, k, r)) yaml_error("expected 'key: value' at line " + std::to_string(lines_[pos_].number));
            ++pos_;
            for (const auto& f : n.fields)
                if (f.first == k) yaml_error("duplicate key '" + k + "'");
            n.fields.emplace_back(k, value_after(r, indent, true));
        }
        if (pos_ < lines_.size() && lines_[pos_].indent > indent)
            yaml_error("bad indentation at line " + std::to_string(lines_[pos_].number));
        return n;
    }

    Node seq_at(int indent) {
        Node n;
        n.kind = Node::Seq;
        while (pos_ < lines_.size() && lines_[pos_].indent == indent && is_item(lines_[pos_])) {
            Line l = lines_[pos_];
            const std::string rest = l.text.size() > 1 ? trim(l.text.substr(1)) : std::string();
            if (rest.empty()) {
                ++pos_;
                n.items.push_back(value_after("", indent, false));
                continue;
            }
            // "- key: v" opens a mapping whose keys sit at indent + offset of rest.
            const int item_indent = indent + static_cast<int>(l.text.find(rest));
            std::string k, r;
            if (split_key(rest, k, r) && rest[0] != '[' && rest[0] != '{') {
                lines_[pos_].indent = item_indent;
                lines_[pos_].text = rest;
                n.items.push_back(map_at(item_indent));
            } else {
                ++pos_;
                n.items.push_back(Flow(rest).parse_all());
            }
        }
        return n;
    }

    std::vector<Line> lines_;
    std::size_t pos_ = 0;
};

Node load_yaml(const std::string& text) {
    std::vector<Line> lines;
    std::size_t start = 0;
    int number = 0;
    while (start <= text.size()) {
        std::size_t end = text.find('\n', start);
        if (end == std::string::npos) end = text.size();
        std::string raw = text.substr(start, end - start);
        ++number;
        start = end + 1;
        if (!raw.empty() && raw.back() == '\r') raw.pop_back();
        if (raw.find('\t') != std::string::npos && raw.find_first_not_of(" \t") != std::string::npos &&
            raw.find('\t') < raw.find_first_not_of(" \t"))
            yaml_error("tabs are not allowed for indentation (line " + std::to_string(number) + ")");
        const std::string t = rtrim(strip_comment(raw));
        if (trim(t).empty() || trim(t) == "---") {
            if (end == text.size()) break;
            continue;
        }
        int ind = 0;
        while (ind < static_cast<int>(t.size()) && t[static_cast<std::size_t>(ind)] == ' ') ++ind;
        lines.push_back({ind, t.substr(static_cast<std::size_t>(ind)), number});
        if (end == text.size()) break;
    }
    return Block(std::move(lines)).parse();
}

// ---- schema ----
[[noreturn]] void bad(const std::string& path, const std::string& what) { fail(ErrorKind::Recipe, path + ": " + what); }

std::string scalar_of(const Node& n, const std::string& path) {
    if (n.kind != Node::Scalar) bad(path, "expected a scalar");
    return n.text;
}

// node.as<int>() of the reference (R/src/recipe.cpp:28-35) goes through yaml-cpp's
// convert<int>::decode: operator>> on a stringstream with std::ios::dec unset, so the
// base comes from the prefix like strtol(.., 0) ("010" is 8, "0x10" is 16, "08" fails),
// an optional sign, no leading whitespace, trailing whitespace allowed, the whole scalar
// consumed, overflow fails. Restated without iostreams (numeric stream extraction is not
// safe in this statically linked libstdc++ once the host process loaded another one).
int int_of(const Node& n, const std::string& path) {
    if (n.kind != Node::Scalar) bad(path, "expected an integer");
    const std::string& s = n.text;
    const auto fail_int = [&] { bad(path, "expected an integer, got '" + s + "'"); };
    std::size_t i = 0;
    bool neg = false;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
    int base = 10;
    if (i + 1 < s.size() && s[i] == '0' && (s[i + 1] == 'x' || s[i + 1] == 'X')) {
        base = 16;
        i += 2;
    } else if (i < s.size() && s[i] == '0') {
        base = 8;
    }
    const std::size_t first = i;
    long long v = 0;
    for (; i < s.size(); ++i) {
        const char c = s[i];
        int d = -1;
        if (c >= '0' && c <= '9') d = c - '0';
        else if (base == 16 && c >= 'a' && c <= 'f') d = c - 'a' + 10;
        else if (base == 16 && c >= 'A' && c <= 'F') d = c - 'A' + 10;
        if (d < 0 || d >= base) break;
        v = v * base + d;
        if (v > 2147483648LL) fail_int();
    }
    if (i == first) fail_int();
    for (; i < s.size(); ++i)
        if (!std::isspace(static_cast<unsigned char>(s[i]))) fail_int();
    if (neg) v = -v;
    if (v < INT32_MIN || v > INT32_MAX) fail_int();
    return static_cast<int>(v);
}

void reject_unknown(const Node& n, const std::set<std::string>& known, const std::string& path) {
    for (const auto& [k, v] : n.fields)
        if (!known.count(k)) bad(path.empty() ? k : path + "." + k, "unknown key");
}

std::vector<int> layers_of(const Node& n, const std::string& path) {
    std::vector<int> out;
    if (n.kind == Node::Seq) {
        for (std::size_t i = 0; i < n.items.size(); ++i) out.push_back(int_of(n.items[i], path + "[" + std::to_string(i) + "]"));
    } else if (n.kind == Node::Map) {
        reject_unknown(n, {"start", "end"}, path);
        const Node* s = n.get("start");
        const Node* e = n.get("end");
        if (!s || !e) bad(path, "range needs both start and end");
        const int a = int_of(*s, path + ".start"), b = int_of(*e, path + ".end");
        if (a < 0 || b <= a) bad(path, "range must satisfy 0 <= start < end");
        for (int i = a; i < b; ++i) out.push_back(i);
    } else {
        bad(path, "expected a list of indices or a {start, end} range");
    }
    for (int l : out)
        if (l < 0) bad(path, "layer indices are 0-based and must be >= 0");
    return out;
}

bool needs_quotes(const std::string& s) {
    if (s.empty()) return true;
    static const std::string kLead = "-?:,[]{}#&*!|>'\"%@` ";
    if (kLead.find(s.front()) != std::string::npos || s.back() == ' ') return true;
    if (s.find(": ") != std::string::npos || s.find(" #") != std::string::npos || s.back() == ':') return true;
    if (s == "~" || s == "null" || s == "true" || s == "false") return true;
    for (char c : s)
        if (c == '\n' || c == '\t' || c == '"') return true;
    return false;
}

std::string yaml_scalar(const std::string& s) {
    if (!needs_quotes(s)) return s;
    std::string out = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') out.push_back('\\');
        if (c == '\n') {
            out += "\\n";
            continue;
        }
        out.push_back(c);
    }
    return out + "\"";
}

std::string flow_ints(const std::vector<int>& v) {
    std::string s = "[";
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + std::to_string(v[i]);
    return s + "]";
}

} // namespace

MergeRecipe parse_recipe(const std::string& yaml_text) {
    const Node root = load_yaml(yaml_text);
    if (root.kind != Node::Map) bad("recipe", "expected a mapping");
    reject_unknown(root, {"merge_method", "base_checkpoint", "num_ranks", "slices", "aux", "config_from"}, "");
    MergeRecipe r;
    const Node* method = root.get("merge_method");
    if (!method) bad("merge_method", "missing (only 'passthrough' is supported)");
    if (const std::string m = scalar_of(*method, "merge_method"); m != "passthrough")
        bad("merge_method", "'" + m + "' is not supported (only 'passthrough')");
    if (const Node* b = root.get("base_checkpoint")) r.base_checkpoint = scalar_of(*b, "base_checkpoint");
    const Node* nr = root.get("num_ranks");
    if (!nr) bad("num_ranks", "missing");
    r.num_ranks = int_of(*nr, "num_ranks");
    if (r.num_ranks < 1) bad("num_ranks", "must be >= 1");
    if (const Node* sl = root.get("slices")) {
        if (sl->kind != Node::Seq) bad("slices", "expected a list");
        for (std::size_t i = 0; i < sl->items.size(); ++i) {
            const std::string path = "slices[" + std::to_string(i) + "]";
            const Node& s = sl->items[i];
            if (s.kind != Node::Map) bad(path, "expected a mapping");
            reject_unknown(s, {"source", "layers", "targets"}, path);
            RecipeSlice slice;
            const Node* src = s.get("source");
            if (!src) bad(path + ".source", "missing");
            slice.source = scalar_of(*src, path + ".source");
            const Node* ly = s.get("layers");
            if (!ly) bad(path + ".layers", "missing");
            slice.layers = layers_of(*ly, path + ".layers");
            if (const Node* t = s.get("targets")) {
                if (t->kind != Node::Seq) bad(path + ".targets", "expected a list");
                for (std::size_t k = 0; k < t->items.size(); ++k)
                    slice.targets.push_back(int_of(t->items[k], path + ".targets[" + std::to_string(k) + "]"));
                if (slice.targets.size() != slice.layers.size()) bad(path + ".targets", "must have the same length as layers");
                for (int l : slice.targets)
                    if (l < 0) bad(path + ".targets", "target indices must be >= 0");
            } else {
                slice.targets = slice.layers;
            }
            r.slices.push_back(std::move(slice));
        }
    }
    if (const Node* aux = root.get("aux")) {
        if (aux->kind != Node::Map) bad("aux", "expected a mapping");
        reject_unknown(*aux, {"embed_tokens", "norm", "lm_head"}, "aux");
        for (const auto& [k, v] : aux->fields) r.aux[k] = scalar_of(v, "aux." + k);
    }
    if (const Node* cf = root.get("config_from")) r.config_from = scalar_of(*cf, "config_from");
    if (r.config_from.empty()) bad("config_from", "must be a path or 'latest'");
    return r;
}

MergeRecipe read_recipe_file(const std::string& path) { return parse_recipe(read_text_file(path)); }

std::string recipe_to_yaml(const MergeRecipe& r) {
    std::string y = "merge_method: passthrough\n";
    if (!r.base_checkpoint.empty()) y += "base_checkpoint: " + yaml_scalar(r.base_checkpoint) + "\n";
    y += "num_ranks: " + std::to_string(r.num_ranks) + "\n";
    if (!r.slices.empty()) {
        y += "slices:\n";
        for (const auto& s : r.slices) {
            y += "  - source: " + yaml_scalar(s.source) + "\n";
            y += "    layers: " + flow_ints(s.layers) + "\n";
            if (s.targets != s.layers) y += "    targets: " + flow_ints(s.targets) + "\n";
        }
    }
    if (!r.aux.empty()) {
        y += "aux:\n";
        for (const char* k : {"embed_tokens", "norm", "lm_head"}) {
            auto it = r.aux.find(k);
            if (it != r.aux.end()) y += std::string("  ") + k + ": " + yaml_scalar(it->second) + "\n";
        }
    }
    y += "config_from: " + yaml_scalar(r.config_from) + "\n";
    return y;
}

} // namespace tailor

// Strict YAML merge-recipe schema (R/src/recipe.cpp:67-169). yaml-cpp is not
// in this image, so this file carries its own YAML reader for what a recipe may be
// written with — block maps and sequences, flow [..] / {..} (also across lines, trailing
// commas), plain scalars (continued on more-indented lines), single- and double-quoted
// scalars (every YAML escape, line folding), block scalars (| and >, chomping and
// indentation indicators), comments, anchors and aliases, tags (which do not change the
// conversions, as in yaml-cpp), %directives, --- / ... markers (the first document, as
// YAML::Load), BOM and CRLF — and an emitter in yaml-cpp's block style. Schema errors
// name the offending field, as the reference's do. tests/test_recipe_yaml.py checks the
// reader against PyYAML on fixed and 600 randomly rendered recipes.
#include <cctype>
#include <cstdint>
#include <map>
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

// &anchor -> node (yaml-cpp resolves *alias to the anchored node)
using Anchors = std::map<std::string, Node>;

[[noreturn]] void yaml_error(const std::string& what) { fail(ErrorKind::Recipe, "invalid YAML: " + what); }

struct Line {
    int indent;
    std::string text; // one logical line: comment-stripped, right-trimmed, continuations folded in
    int number;
};

bool is_ws(char c) { return c == ' ' || c == '\t'; }

std::string rtrim(std::string s) {
    while (!s.empty() && std::isspace(static_cast<unsigned char>(s.back()))) s.pop_back();
    return s;
}

std::string trim(const std::string& s) {
    std::size_t b = 0;
    while (b < s.size() && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
    return rtrim(s.substr(b));
}

// A quote (or a flow bracket) opens a node only where a node starts; elsewhere ' " [ {
// are plain characters ("/runs/bob's/ck-100", "/data/[v2]"). In block context (depth 0)
// a node starts at the line start or after "- ", ": ", "? "; inside a flow collection
// also after "[", "{", ",".
bool node_starts(const std::string& s, std::size_t i, int depth) {
    std::size_t j = i;
    while (j > 0 && is_ws(s[j - 1])) --j;
    if (j == 0) return true;
    const char p = s[j - 1];
    if (depth > 0 && (p == '[' || p == '{' || p == ',')) return true;
    return (p == ':' || p == '-' || p == '?') && j < i && (j == 1 || depth > 0 || p != '-' || is_ws(s[j - 2])); // "key: 'v'", "- 'v'"
}

// Scans s from state (quote, depth): returns where a comment starts (npos if none) and
// leaves the quote / flow-bracket state at the end of the line.
std::size_t scan(const std::string& s, char& quote, int& depth) {
    for (std::size_t i = 0; i < s.size(); ++i) {
        const char c = s[i];
        if (quote) {
            if (quote == '"' && c == '\\') {
                ++i;
                continue;
            }
            if (c == quote) {
                if (quote == '\'' && i + 1 < s.size() && s[i + 1] == '\'') {
                    ++i;
                    continue;
                }
                quote = 0;
            }
            continue;
        }
        if ((c == '"' || c == '\'') && node_starts(s, i, depth)) quote = c;
        else if (c == '#' && (i == 0 || is_ws(s[i - 1]))) return i;
        else if ((c == '[' || c == '{') && (depth > 0 || node_starts(s, i, 0))) ++depth; // mid-scalar brackets are plain text
        else if ((c == ']' || c == '}') && depth > 0) --depth;
    }
    return std::string::npos;
}

std::string strip_comment(const std::string& s) {
    char q = 0;
    int d = 0;
    const std::size_t at = scan(s, q, d);
    return at == std::string::npos ? s : s.substr(0, at);
}

void put_utf8(std::string& o, std::uint32_t cp) {
    if (cp < 0x80) {
        o.push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
        o.push_back(static_cast<char>(0xC0 | (cp >> 6)));
        o.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
        o.push_back(static_cast<char>(0xE0 | (cp >> 12)));
        o.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
        o.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x110000) {
        o.push_back(static_cast<char>(0xF0 | (cp >> 18)));
        o.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
        o.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
        o.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
        yaml_error("escaped code point out of range");
    }
}

// A double-quoted scalar's content as yaml-cpp writes it (used for folded block scalars).
std::string dq(const std::string& v) {
    std::string o = "\"";
    for (const char c : v) {
        if (c == '"' || c == '\\') {
            o.push_back('\\');
            o.push_back(c);
        } else if (c == '\n') {
            o += "\\n";
        } else if (c == '\t') {
            o += "\\t";
        } else if (static_cast<unsigned char>(c) < 0x20) {
            static const char* hx = "0123456789abcdef";
            o += "\\x";
            o.push_back(hx[(c >> 4) & 0xF]);
            o.push_back(hx[c & 0xF]);
        } else {
            o.push_back(c);
        }
    }
    return o + "\"";
}

// ---- flow / scalar parsing ----
class Flow {
  public:
    Flow(const std::string& s, Anchors& anchors) : s_(s), anchors_(anchors) {}
    Node parse_all() {
        Node n = value(false);
        ws();
        if (i_ != s_.size()) yaml_error("unexpected trailing text '" + s_.substr(i_) + "'");
        return n;
    }

  private:
    void ws() {
        while (i_ < s_.size() && is_ws(s_[i_])) ++i_;
    }
    bool at_end_of_node(bool in_flow) const {
        return i_ >= s_.size() || (in_flow && (s_[i_] == ',' || s_[i_] == ']' || s_[i_] == '}'));
    }
    std::string token() { // anchor / alias / tag name: up to whitespace or a flow indicator
        const std::size_t b = i_;
        while (i_ < s_.size() && !is_ws(s_[i_]) && s_[i_] != ',' && s_[i_] != '[' && s_[i_] != ']' && s_[i_] != '{' &&
               s_[i_] != '}')
            ++i_;
        return s_.substr(b, i_ - b);
    }
    Node value(bool in_flow) {
        ws();
        std::string anchor;
        while (i_ < s_.size() && (s_[i_] == '&' || s_[i_] == '!')) { // node properties; tags do not change conversions
            const bool is_anchor = s_[i_] == '&';
            ++i_;
            const std::string name = token();
            if (is_anchor) {
                if (name.empty()) yaml_error("empty anchor name");
                anchor = name;
            }
            ws();
        }
        Node n;
        if (i_ < s_.size() && s_[i_] == '*') {
            if (!anchor.empty()) yaml_error("an alias cannot carry an anchor");
            ++i_;
            const std::string name = token();
            const auto it = anchors_.find(name);
            if (it == anchors_.end()) yaml_error("unknown anchor '" + name + "'");
            return it->second;
        }
        if (at_end_of_node(in_flow)) n = Node{};
        else if (s_[i_] == '[') n = seq();
        else if (s_[i_] == '{') n = map();
        else n = scalar(in_flow, false);
        if (!anchor.empty()) anchors_[anchor] = n;
        return n;
    }
    void escape(std::string& out) {
        if (i_ >= s_.size()) yaml_error("bad escape");
        const char e = s_[i_++];
        const auto hex = [&](int digits) {
            std::uint32_t v = 0;
            for (int k = 0; k < digits; ++k) {
                if (i_ >= s_.size() || !std::isxdigit(static_cast<unsigned char>(s_[i_]))) yaml_error("bad escape");
                const char h = s_[i_++];
                v = v * 16 + static_cast<std::uint32_t>(std::isdigit(static_cast<unsigned char>(h)) ? h - '0' : (std::tolower(h) - 'a' + 10));
            }
            return v;
        };
        switch (e) {
            case '0': out.push_back('\0'); break;
            case 'a': out.push_back('\a'); break;
            case 'b': out.push_back('\b'); break;
            case 't': case '\t': out.push_back('\t'); break;
            case 'n': out.push_back('\n'); break;
            case 'v': out.push_back('\v'); break;
            case 'f': out.push_back('\f'); break;
            case 'r': out.push_back('\r'); break;
            case 'e': out.push_back('\x1b'); break;
            case ' ': case '"': case '/': case '\\': out.push_back(e); break;
            case 'N': put_utf8(out, 0x85); break;
            case '_': put_utf8(out, 0xA0); break;
            case 'L': put_utf8(out, 0x2028); break;
            case 'P': put_utf8(out, 0x2029); break;
            case 'x': put_utf8(out, hex(2)); break;
            case 'u': put_utf8(out, hex(4)); break;
            case 'U': put_utf8(out, hex(8)); break;
            default: yaml_error(std::string("unknown escape character '") + e + "'");
        }
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
                    escape(n.text);
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
            if (is_key && c == ':' && (i_ + 1 == s_.size() || is_ws(s_[i_ + 1]) || (in_flow && (s_[i_ + 1] == ',' || s_[i_ + 1] == '}'))))
                break;
            ++i_;
        }
        n.text = trim(s_.substr(b, i_ - b));
        if (n.text.empty() || n.text == "~" || n.text == "null" || n.text == "Null" || n.text == "NULL") {
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
                ws();
                if (i_ < s_.size() && s_[i_] == ']') { // trailing comma
                    ++i_;
                    return n;
                }
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
                ws();
                if (i_ < s_.size() && s_[i_] == '}') { // trailing comma
                    ++i_;
                    return n;
                }
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
    Anchors& anchors_;
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
            if (quote == '"' && c == '\\') {
                ++i;
                continue;
            }
            if (c == quote) {
                if (quote == '\'' && i + 1 < t.size() && t[i + 1] == '\'') {
                    ++i;
                    continue;
                }
                quote = 0;
            }
            continue;
        }
        if ((c == '"' || c == '\'') && node_starts(t, i, depth)) quote = c;
        else if ((c == '[' || c == '{') && (depth > 0 || node_starts(t, i, 0))) ++depth;
        else if ((c == ']' || c == '}') && depth > 0) --depth;
        else if (c == ':' && depth == 0 && (i + 1 == t.size() || is_ws(t[i + 1]))) {
            std::string k = trim(t.substr(0, i));
            if (k.size() >= 2 && (k.front() == '"' || k.front() == '\'') && k.back() == k.front()) {
                Anchors none;
                k = Flow(k, none).parse_all().text; // quoted keys: escapes and '' resolved
            }
            key = k;
            rest = trim(t.substr(i + 1));
            return !key.empty();
        }
    }
    return false;
}

// Leading node properties of a block value ("&a !!map"): returns the anchor (if any) and
// strips them from `rest`.
std::string take_properties(std::string& rest) {
    std::string anchor;
    while (!rest.empty() && (rest[0] == '&' || rest[0] == '!')) {
        std::size_t e = 0;
        while (e < rest.size() && !is_ws(rest[e])) ++e;
        if (rest[0] == '&') anchor = rest.substr(1, e - 1);
        rest = trim(rest.substr(e));
    }
    return anchor;
}

class Block {
  public:
    Block(std::vector<Line> lines, Anchors& anchors) : lines_(std::move(lines)), anchors_(anchors) {}
    Node parse() {
        if (lines_.empty()) return Node{};
        Node n = node_at(lines_[0].indent);
        if (pos_ != lines_.size()) yaml_error("unexpected content at line " + std::to_string(lines_[pos_].number));
        return n;
    }

  private:
    bool is_item(const Line& l) const { return l.text == "-" || l.text.rfind("- ", 0) == 0 || l.text.rfind("-\t", 0) == 0; }

    Node flow(const std::string& s) { return Flow(s, anchors_).parse_all(); }

    Node node_at(int indent) {
        const Line& l = lines_[pos_];
        if (l.indent != indent) yaml_error("bad indentation at line " + std::to_string(l.number));
        if (is_item(l)) return seq_at(indent);
        std::string k, r;
        if (split_key(l.text, k, r)) return map_at(indent);
        ++pos_;
        return flow(l.text);
    }

    Node value_after(std::string rest, int indent, bool allow_same_indent_seq) {
        const std::string anchor = take_properties(rest);
        Node n;
        if (!rest.empty()) {
            n = flow(rest);
        } else if (pos_ < lines_.size()) {
            const Line& nx = lines_[pos_];
            if (nx.indent > indent) n = node_at(nx.indent);
            else if (allow_same_indent_seq && nx.indent == indent && is_item(nx)) n = seq_at(indent);
        }
        if (!anchor.empty()) anchors_[anchor] = n;
        return n;
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
            std::string rest = l.text.size() > 1 ? trim(l.text.substr(1)) : std::string();
            const std::string anchor = take_properties(rest);
            if (rest.empty()) {
                ++pos_;
                Node v = value_after("", indent, false);
                if (!anchor.empty()) anchors_[anchor] = v;
                n.items.push_back(std::move(v));
                continue;
            }
            // "- key: v" opens a mapping whose keys sit at indent + offset of rest.
            const int item_indent = indent + static_cast<int>(l.text.rfind(rest));
            std::string k, r;
            Node v;
            if (split_key(rest, k, r) && rest[0] != '[' && rest[0] != '{') {
                lines_[pos_].indent = item_indent;
                lines_[pos_].text = rest;
                v = map_at(item_indent);
            } else {
                ++pos_;
                v = flow(rest);
            }
            if (!anchor.empty()) anchors_[anchor] = v;
            n.items.push_back(std::move(v));
        }
        return n;
    }

    std::vector<Line> lines_;
    Anchors& anchors_;
    std::size_t pos_ = 0;
};

int indent_of(const std::string& raw) {
    int ind = 0;
    while (ind < static_cast<int>(raw.size()) && raw[static_cast<std::size_t>(ind)] == ' ') ++ind;
    return ind;
}

bool blank(const std::string& raw) { return raw.find_first_not_of(" \t") == std::string::npos; }

// Column of the node a logical line's value belongs to: the indent plus any "- " item
// prefixes and, for "key: value", the key's column (block scalars and plain-scalar
// continuation lines must be indented beyond it).
int owner_column(const Line& l) {
    std::size_t i = 0, dash = std::string::npos;
    while (i + 1 < l.text.size() && l.text[i] == '-' && is_ws(l.text[i + 1])) {
        dash = i;
        i += 2;
        while (i < l.text.size() && is_ws(l.text[i])) ++i;
    }
    std::string k, r;
    if (dash != std::string::npos && !split_key(l.text.substr(i), k, r)) // "- value": the item's dash
        return l.indent + static_cast<int>(dash);
    return l.indent + static_cast<int>(i); // "key: value" / "- key: value": the key
}

// The value part of a logical line ("key: v" -> v, "- v" -> v), after properties.
std::string value_part(const std::string& body) {
    std::string t = body;
    while (t.size() >= 2 && t[0] == '-' && is_ws(t[1])) t = trim(t.substr(2));
    if (t == "-") return "";
    std::string k, r;
    if (t.empty() || t[0] == '[' || t[0] == '{' || t[0] == '"' || t[0] == '\'') return t;
    if (split_key(t, k, r)) t = r;
    take_properties(t);
    return t;
}

bool block_indicator(const std::string& v, char& style, char& chomp, int& explicit_indent) {
    if (v.empty() || (v[0] != '|' && v[0] != '>')) return false;
    style = v[0];
    chomp = 0;
    explicit_indent = 0;
    for (std::size_t i = 1; i < v.size(); ++i) {
        const char c = v[i];
        if ((c == '+' || c == '-') && !chomp) chomp = c;
        else if (c >= '1' && c <= '9' && !explicit_indent) explicit_indent = c - '0';
        else return false;
    }
    return true;
}

// Splits the document into logical lines: BOM, directives and document markers handled
// (yaml-cpp's Load reads the first document), comments stripped, quoted scalars and flow
// collections that span lines joined, plain scalars' continuation lines folded, block
// scalars (| and >, chomping and indentation indicators) turned into one double-quoted
// scalar. The Block parser then sees one line per node.
std::vector<Line> logical_lines(const std::string& text_in) {
    std::string text = text_in;
    if (text.rfind("\xEF\xBB\xBF", 0) == 0) text = text.substr(3);
    std::vector<std::string> raw;
    for (std::size_t start = 0; start <= text.size();) {
        std::size_t end = text.find('\n', start);
        if (end == std::string::npos) end = text.size();
        std::string r = text.substr(start, end - start);
        if (!r.empty() && r.back() == '\r') r.pop_back();
        raw.push_back(std::move(r));
        if (end == text.size()) break;
        start = end + 1;
    }
    std::vector<Line> out;
    bool content = false, in_doc = false;
    for (std::size_t i = 0; i < raw.size(); ++i) {
        std::string r = raw[i];
        const int number = static_cast<int>(i) + 1;
        const auto marker_in = [](const std::string& x, const char* m) { return x.rfind(m, 0) == 0 && (x.size() == 3 || is_ws(x[3])); };
        const auto marker = [&](const char* m) { return marker_in(r, m); };
        if (!content && !in_doc && !r.empty() && r[0] == '%') continue; // directive
        if (marker("---")) {
            if (content || in_doc) break; // a second document
            in_doc = true;
            r = r.substr(3);
            if (blank(strip_comment(r))) continue;
            r = trim(r); // "--- value" on the marker line
        } else if (marker("...")) {
            break;
        }
        if (!blank(r) && r.find('\t') < r.find_first_not_of(" \t"))
            yaml_error("tabs are not allowed for indentation (line " + std::to_string(number) + ")");
        char q = 0;
        int depth = 0;
        std::size_t cut = scan(r, q, depth);
        std::string logical = cut == std::string::npos ? r : r.substr(0, cut);
        if (blank(logical) && !q) continue;
        const int indent = indent_of(logical);
        // quoted scalars and flow collections continued on the next lines
        int pending_breaks = 0;
        while ((q || depth > 0) && i + 1 < raw.size()) {
            const std::string nl = raw[++i];
            if (marker_in(nl, "---") || marker_in(nl, "...")) yaml_error("document marker inside a flow or quoted node");
            if (q) {
                std::string c = trim(nl);
                if (c.empty()) {
                    ++pending_breaks;
                    continue;
                }
                std::string head = logical;
                while (!head.empty() && is_ws(head.back())) head.pop_back();
                std::size_t bs = 0; // an odd run of trailing backslashes escapes the line break
                while (bs < head.size() && head[head.size() - 1 - bs] == '\\') ++bs;
                if (q == '"' && bs % 2 == 1 && !pending_breaks) {
                    head.pop_back();
                    logical = head;
                } else {
                    logical = head + (pending_breaks ? std::string(static_cast<std::size_t>(pending_breaks), '\n') : std::string(" "));
                }
                pending_breaks = 0;
                cut = scan(c, q, depth);
                logical += cut == std::string::npos ? c : c.substr(0, cut);
            } else {
                std::string c = trim(nl);
                cut = scan(c, q, depth);
                logical += " " + (cut == std::string::npos ? c : c.substr(0, cut));
            }
        }
        if (q) yaml_error("unterminated quoted scalar starting at line " + std::to_string(number));
        if (depth > 0) yaml_error("unterminated flow collection starting at line " + std::to_string(number));
        Line l{indent, rtrim(logical.substr(static_cast<std::size_t>(indent))), number};
        const int owner = owner_column(l);
        const std::string v = value_part(l.text);
        char style = 0, chomp = 0;
        int ind = 0;
        if (block_indicator(v, style, chomp, ind)) {
            // block scalar: the following lines indented beyond the owner (and blank lines)
            std::vector<std::string> body;
            int content_indent = ind ? owner + ind : -1;
            while (i + 1 < raw.size()) {
                const std::string& nl = raw[i + 1];
                if (blank(nl)) {
                    body.push_back(nl);
                    ++i;
                    continue;
                }
                const int ni = indent_of(nl);
                if (content_indent < 0) {
                    if (ni <= owner) break;
                    content_indent = ni;
                }
                if (ni < content_indent) break;
                body.push_back(nl);
                ++i;
            }
            if (content_indent < 0) content_indent = owner + 1;
            // trailing blank lines belong to the chomping, not the content
            std::size_t last = body.size();
            while (last > 0 && blank(body[last - 1])) --last;
            std::vector<std::string> ls;
            for (std::size_t k = 0; k < last; ++k)
                ls.push_back(static_cast<int>(body[k].size()) > content_indent ? body[k].substr(static_cast<std::size_t>(content_indent)) : std::string());
            std::string val;
            if (style == '|') {
                for (std::size_t k = 0; k < ls.size(); ++k) val += (k ? "\n" : "") + ls[k];
            } else {
                int empties = 0;
                bool have = false, prev_more = false;
                for (const auto& x : ls) {
                    if (x.empty()) {
                        ++empties;
                        continue;
                    }
                    const bool more = is_ws(x[0]);
                    if (have) val += empties ? std::string(static_cast<std::size_t>(empties) + ((prev_more || more) ? 1 : 0), '\n')
                                             : std::string((prev_more || more) ? "\n" : " ");
                    else if (empties) val += std::string(static_cast<std::size_t>(empties), '\n');
                    val += x;
                    have = true;
                    prev_more = more;
                    empties = 0;
                }
            }
            if (chomp == '-') {
                // strip: no trailing line break
            } else if (chomp == '+') {
                if (!ls.empty()) val += "\n";
                for (std::size_t k = last; k < body.size(); ++k) val += "\n";
            } else if (!ls.empty()) {
                val += "\n";
            }
            const std::size_t at = l.text.rfind(v);
            l.text = l.text.substr(0, at) + dq(val);
        } else if (!v.empty() && v[0] != '[' && v[0] != '{' && v[0] != '"' && v[0] != '\'' && v[0] != '*') {
            // plain scalar: more-indented lines that follow continue it (folded with spaces)
            int breaks = 0;
            std::string extra;
            while (i + 1 < raw.size()) {
                const std::string& nl = raw[i + 1];
                const std::string c = rtrim(strip_comment(nl));
                if (blank(c)) {
                    if (!blank(nl)) break; // a comment line ends a plain scalar
                    ++breaks;
                    ++i;
                    continue;
                }
                if (indent_of(nl) <= owner || trim(nl).rfind("#", 0) == 0) break;
                extra += breaks ? std::string(static_cast<std::size_t>(breaks), '\n') : std::string(" ");
                extra += trim(c);
                breaks = 0;
                ++i;
            }
            if (!extra.empty()) {
                const std::size_t at = l.text.rfind(v);
                l.text = l.text.substr(0, at) + dq(v + extra);
            }
        }
        content = true;
        out.push_back(std::move(l));
    }
    return out;
}

Node load_yaml(const std::string& text) {
    Anchors anchors;
    return Block(logical_lines(text), anchors).parse();
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

"""Recipe YAML coverage. The reference parses recipes with yaml-cpp (R/src/recipe.cpp:67-132),
an external dependency this image lacks; the library carries its own reader
(csrc/host/recipe.cpp). These tests render the same recipes in the YAML styles a user or a
tool may write — block and flow collections (also spanning lines), plain / single / double
quoted scalars (escapes, folding), block scalars (| and > with chomping), comments, anchors
and aliases, tags, document markers and directives, BOM, CRLF — and check the parse
against PyYAML's reading of the same text (the structural oracle: both are YAML readers;
the cases avoid the YAML 1.1 scalar forms where PyYAML and yaml-cpp differ, e.g. yes/no
and 010)."""
import json
import random

import pytest

yaml = pytest.importorskip("yaml")

import paper_2602_22158_b200 as t  # noqa: E402


def expected(doc):
    """The reference's schema applied to an already-parsed document (R/src/recipe.cpp:67-132)."""
    slices = []
    for s in doc.get("slices") or []:
        ly = s["layers"]
        layers = list(range(ly["start"], ly["end"])) if isinstance(ly, dict) else list(ly)
        slices.append({"source": s["source"], "layers": layers, "targets": list(s.get("targets", layers))})
    return {"base_checkpoint": doc.get("base_checkpoint", ""), "num_ranks": doc["num_ranks"], "slices": slices,
            "aux": dict(doc.get("aux") or {}), "config_from": doc.get("config_from", "latest")}


def ours(text):
    return json.loads(t.parse_recipe(text).to_json())


def check(text):
    want = expected(yaml.safe_load(text))
    got = ours(text)
    assert got == want, text


CASES = {
    "block": "merge_method: passthrough\nnum_ranks: 2\nslices:\n  - source: /a/ck-100\n    layers: [0, 1]\n"
             "  - source: /a/ck-200\n    layers: {start: 2, end: 4}\naux:\n  embed_tokens: /a/ck-100\n",
    "flow_items": "merge_method: passthrough\nnum_ranks: 2\nslices:\n  - {source: /a/ck-100, layers: [0, 1]}\n"
                  "  - {source: \"/a/ck-200\", layers: {start: 2, end: 4}, targets: [2, 3]}\n",
    "markers_comments": "--- # recipe\nmerge_method: passthrough   # only one\nnum_ranks: 2\n# a comment line\n"
                        "slices:\n- source: '/a/ck-100'\n  layers:\n    - 0\n    - 1\n...\n",
    "multiline_flow": "merge_method: passthrough\nnum_ranks: 2\nslices: [\n  {source: /a/ck-100, layers: [0,\n     1]},\n]\n",
    "anchors": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: &b /a/ck-300\naux:\n  norm: *b\n",
    "whole_flow": "{merge_method: passthrough, num_ranks: 2, base_checkpoint: /a/ck-1}",
    "tags": "merge_method: !!str passthrough\nnum_ranks: !!int 2\nbase_checkpoint: /a/ck-1\n",
    "crlf": "merge_method: passthrough\r\nnum_ranks: 2\r\nbase_checkpoint: /a/ck-1\r\n",
    "escapes": 'merge_method: "passthrough"\nnum_ranks: 2\nbase_checkpoint: "/a/ck\\u002d1\\x41\\t\\\\"\n',
    "plain_continued": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: /a/very\n  long\n",
    "folded": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: >-\n  /a/ck-1\n",
    "literal_clip": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: |-\n  /a/ck-1\nconfig_from: |\n  latest\n",
    "literal_keep": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: |+\n  /a/ck-1\n\nconfig_from: x\n",
    "folded_paragraphs": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: >\n  a\n  b\n\n  c\n",
    "bom": "\ufeffmerge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: /a/ck-1\n",
    "apostrophe_plain": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: /runs/bob's/ck-1 # note\n",
    "multiline_quoted": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: \"/a/ck\\\n  -1\"\naux: {norm: 'x\n  y'}\n",
    "quoted_blank_line": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: \"a\n\n  b\"\n",
    "anchor_map": "merge_method: passthrough\nnum_ranks: 2\nslices:\n  - &s\n    source: /a/ck-1\n    layers: [0]\n  - *s\n",
    "anchor_seq": "merge_method: passthrough\nnum_ranks: 2\nslices:\n  - source: /a/ck-1\n    layers: &l [0, 1]\n"
                  "  - source: /a/ck-2\n    layers: *l\n    targets: *l\n",
    "directive": "%YAML 1.2\n---\nmerge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: /a/ck-1\n",
    "trailing_comma": "merge_method: passthrough\nnum_ranks: 2\nslices: [{source: a, layers: [0, 1,],},]\n",
    "quoted_keys": "\"merge_method\": passthrough\n'num_ranks': 2\nbase_checkpoint: /a/ck-1\n",
    "hash_in_plain": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: /a/ck#1\n",
    "url_like": "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: s3://bucket/ck-1\n",
    "item_block_scalar": "merge_method: passthrough\nnum_ranks: 2\nslices:\n- source: |-\n    /a/ck-1\n  layers:\n  - 3\n"
                         "aux:\n  norm:\n    >-\n     x\n",
    "item_plain_continued": "merge_method: passthrough\nnum_ranks: 2\nslices:\n- source: /a/ck\n    -1\n  layers: [0]\n"
                            "aux:\n  norm: x\n    y\n",
    "seq_item_scalars": "merge_method: passthrough\nnum_ranks: 2\nslices:\n- source: a\n  layers:\n  - 1\n  - 2\n"
                        "aux:\n  norm: >-\n   a\n   b\n",
    "indentless_range": "merge_method: passthrough\nnum_ranks: 2\nslices:\n- source: /a/ck-100\n  layers:\n    start: 0\n    end: 2\n",
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_yaml_styles_parse_like_a_yaml_reader(name):
    check(CASES[name])


def test_integers_from_any_scalar_style_like_yaml_cpp():
    """yaml-cpp's as<int>() converts the scalar's text whatever its style (PyYAML would
    keep a quoted or block scalar a string), R/src/recipe.cpp:28-35."""
    text = "merge_method: passthrough\nnum_ranks: '2'\nslices:\n- source: a\n  layers:\n  - |-\n    1\n  - \"2\"\n"
    got = ours(text)
    assert got["num_ranks"] == 2 and got["slices"][0]["layers"] == [1, 2]


def test_first_document_only_like_yaml_cpp_load():
    text = "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: /a/ck-1\n---\nfoo: 1\n"
    assert ours(text)["base_checkpoint"] == "/a/ck-1"


@pytest.mark.parametrize("text", [
    "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: *nope\n",         # unknown alias
    "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: \"/a\\q\"\n",     # unknown escape
    "merge_method: passthrough\nnum_ranks: 2\nslices: [\n  {source: a, layers: [0]}\n",  # unterminated flow
    "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: \"abc\n",         # unterminated quote
    "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: ~\n",             # null is not a scalar
    "merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: NULL\n",
    "merge_method: passthrough\nnum_ranks: 2\nslices: [\n---\n]\n",             # marker inside a flow node
])
def test_malformed_or_null_are_recipe_errors(text):
    with pytest.raises(t.TailorError) as e:
        t.parse_recipe(text)
    assert e.value.kind == t.ErrorKind.Recipe


# ---- randomized renderings of random recipes ------------------------------------------------
def _plain_ok(s):
    return all(c.isalnum() or c in "/-_.@" for c in s) and not s[0] in "-@"


def _scalar(rng, s, indent):
    """One rendering of string s: plain, single-quoted, double-quoted (with escapes), or a
    block scalar (only where a block value may start)."""
    k = rng.randrange(6)
    if k == 0 and _plain_ok(s):
        return s
    if k == 5 and indent is not None and " " in s and _plain_ok(s.replace(" ", "")):
        return s.replace(" ", "\n" + " " * (indent + 2), 1)  # plain scalar continued (folded to a space)
    if k == 1:
        return "'" + s.replace("'", "''") + "'"
    if k == 2:
        out = []
        for c in s:
            r = rng.random()
            if c in '"\\':
                out.append("\\" + c)
            elif r < 0.1:
                out.append("\\x%02x" % ord(c))
            elif r < 0.2:
                out.append("\\u%04x" % ord(c))
            else:
                out.append(c)
        return '"' + "".join(out) + '"'
    if k == 3 and indent is not None:
        return "|-\n" + " " * (indent + 2) + s
    if k == 4 and indent is not None:
        return ">-\n" + " " * (indent + 2) + s
    return '"' + s.replace("\\", "\\\\").replace('"', '\\"') + '"'


def _ints(rng, xs, indent):
    if rng.random() < 0.5 or indent is None:
        sep = rng.choice([", ", ",", " ,  "])
        body = sep.join(str(x) for x in xs)
        if rng.random() < 0.3 and len(xs) > 1:  # spread over lines
            body = (",\n" + " " * (indent or 0) + "  ").join(str(x) for x in xs)
        return "[" + body + (rng.choice(["", ","]) if xs else "") + "]"
    return "\n" + "".join(" " * (indent + 2) + "- " + str(x) + "\n" for x in xs).rstrip("\n")


def render(rng, rec):
    lines = []
    if rng.random() < 0.2:
        lines.append("%YAML 1.2")
        lines.append("---")
    elif rng.random() < 0.3:
        lines.append("--- # recipe")
    anchors = {}
    keys = ["merge_method", "num_ranks", "base_checkpoint", "slices", "aux", "config_from"]
    rng.shuffle(keys)

    def src(s, indent, inline=False):
        if s in anchors and rng.random() < 0.5:
            return "*" + anchors[s]
        v = _scalar(rng, s, None if inline else indent)
        if s not in anchors and rng.random() < 0.3 and not v.startswith(("|", ">")):
            anchors[s] = "a%d" % len(anchors)
            return "&" + anchors[s] + " " + v
        return v

    for k in keys:
        if rng.random() < 0.15:
            lines.append("# " + k)
        if k == "merge_method":
            lines.append("merge_method: " + rng.choice(["passthrough", "'passthrough'", '"passthrough"', "!!str passthrough"]))
        elif k == "num_ranks":
            lines.append("num_ranks: " + rng.choice([str(rec["num_ranks"]), "!!int %d" % rec["num_ranks"]])
                         + rng.choice(["", "  # ranks"]))
        elif k == "base_checkpoint" and rec["base_checkpoint"]:
            lines.append("base_checkpoint: " + src(rec["base_checkpoint"], 0))
        elif k == "config_from" and rec["config_from"] != "latest":
            lines.append("config_from: " + src(rec["config_from"], 0))
        elif k == "aux" and rec["aux"]:
            if rng.random() < 0.4:
                lines.append("aux: {" + ", ".join(f"{m}: {src(v, 0, True)}" for m, v in rec["aux"].items()) + "}")
            else:
                lines.append("aux:")
                for m, v in rec["aux"].items():
                    lines.append(f"  {m}: " + src(v, 2))
        elif k == "slices" and rec["slices"]:
            if rng.random() < 0.25:
                items = []
                for s in rec["slices"]:
                    items.append("{source: " + src(s["source"], 0, True) + ", layers: " + _ints(rng, s["layers"], None)
                                 + ", targets: " + _ints(rng, s["targets"], None) + "}")
                lines.append("slices: [" + (",\n  ".join(items) if rng.random() < 0.5 else ", ".join(items)) + "]")
            else:
                lines.append("slices:")
                ind = rng.choice([0, 2, 4])
                for s in rec["slices"]:
                    lines.append(" " * ind + "- source: " + src(s["source"], ind + 2))
                    lr = s["layers"]
                    contiguous = lr == list(range(lr[0], lr[-1] + 1))
                    if contiguous and rng.random() < 0.4:
                        if rng.random() < 0.5:
                            lines.append(" " * (ind + 2) + f"layers: {{start: {lr[0]}, end: {lr[-1] + 1}}}")
                        else:
                            lines.append(" " * (ind + 2) + "layers:")
                            lines.append(" " * (ind + 4) + f"start: {lr[0]}")
                            lines.append(" " * (ind + 4) + f"end: {lr[-1] + 1}")
                    else:
                        lines.append(" " * (ind + 2) + "layers: " + _ints(rng, lr, ind + 2))
                    lines.append(" " * (ind + 2) + "targets: " + _ints(rng, s["targets"], ind + 2))
    if rng.random() < 0.2:
        lines.append("...")
    eol = "\r\n" if rng.random() < 0.1 else "\n"
    return ("\ufeff" if rng.random() < 0.05 else "") + eol.join(lines) + eol


def random_recipe(rng):
    paths = ["/runs/r%d/checkpoint-%d" % (rng.randrange(3), 100 * rng.randrange(1, 9)) for _ in range(4)]
    paths += ["/runs/bob's run/ck-1", "s3://b/k#1", "C:/x y/ck", "ck-\u00e9"]
    L = rng.randrange(1, 9)
    slices, free = [], list(range(L))
    rng.shuffle(free)
    while free and rng.random() < 0.8:
        n = rng.randrange(1, len(free) + 1)
        ls = sorted(free[:n]) if rng.random() < 0.5 else free[:n]
        free = free[n:]
        slices.append({"source": rng.choice(paths), "layers": ls, "targets": ls})
    aux = {m: rng.choice(paths) for m in ("embed_tokens", "norm", "lm_head") if rng.random() < 0.5}
    return {"base_checkpoint": rng.choice(paths) if rng.random() < 0.5 else "", "num_ranks": rng.randrange(1, 9),
            "slices": slices, "aux": aux, "config_from": rng.choice(["latest", "latest", rng.choice(paths)])}


def test_random_renderings_parse_like_a_yaml_reader():
    rng = random.Random(2602)
    for case in range(600):
        rec = random_recipe(rng)
        text = render(rng, rec)
        doc = yaml.safe_load(text.lstrip("\ufeff"))
        assert expected(doc) == rec, (case, text)  # the rendering itself is right
        assert ours(text) == rec, (case, text)


def test_emitter_round_trips_awkward_strings():
    """recipe_to_yaml quotes what a YAML reader would not read back as the same string
    (indicators, brackets, quotes, '#', ': ', tabs, newlines, unicode): our reader and
    PyYAML both recover every string."""
    rng = random.Random(7)
    alphabet = list("abcXYZ019/-_.:#&*!|>'\"%@`,[]{}? \t\\é✓") + ["\n"]
    for _ in range(3000):
        s = "".join(rng.choice(alphabet) for _ in range(rng.randrange(1, 12)))
        rec = t.MergeRecipe(num_ranks=2, base_checkpoint=s, aux={"norm": s})
        y = rec.to_yaml()
        assert t.parse_recipe(y) == rec, y
        d = yaml.safe_load(y)
        assert str(d["aux"]["norm"]) == s or isinstance(d["aux"]["norm"], (int, float)), y  # 1.1 typing of "9"


@pytest.mark.parametrize("text,value", [
    ("base_checkpoint: /data/[v2]/ck\n", "/data/[v2]/ck"),
    ("base_checkpoint: a{b'c\n", "a{b'c"),
    ("base_checkpoint: x-'y'\n", "x-'y'"),
    ("base_checkpoint: /p/[[x\n", "/p/[[x"),
])
def test_brackets_and_quotes_inside_plain_scalars_are_text(text, value):
    assert ours("merge_method: passthrough\nnum_ranks: 2\n" + text)["base_checkpoint"] == value

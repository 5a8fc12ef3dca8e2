// table_io.cpp -- transition-table text I/O (host only).
//
// "During this transformation, the PaREM creates a log file with the transition table"
// (P:314).  The format is SPEC's, UTF-8 / LF:
//     symbols<TAB>s1<TAB>s2...      one character per symbol
//     start<TAB><id>
//     finals[<TAB><id>...]          zero or more ids
//     <state-id><TAB><dest or ->... one row per state in id order, '-' = DEAD
// A symbol that is not a printable ASCII character other than backslash is written \xHH.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "internal.h"

using namespace parem;

namespace {

void put_symbol(std::string& o, unsigned char c) {
    if (c > 0x20 && c < 0x7F && c != '\\') {
        o.push_back((char)c);
    } else {
        char b[8];
        snprintf(b, sizeof(b), "\\x%02X", c);
        o += b;
    }
}

struct Lines {
    const char* p;
    const char* end;
    uint32_t line = 0;
    // next line without its LF (and a trailing CR); false at the end of the text
    bool next(std::string& out) {
        if (p >= end) return false;
        const char* q = (const char*)memchr(p, '\n', (size_t)(end - p));
        const char* e = q ? q : end;
        out.assign(p, e);
        if (!out.empty() && out.back() == '\r') out.pop_back();
        p = q ? q + 1 : end;
        ++line;
        return true;
    }
};

std::vector<std::string> split_tabs(const std::string& s) {
    std::vector<std::string> f;
    size_t a = 0;
    for (;;) {
        const size_t b = s.find('\t', a);
        f.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
        if (b == std::string::npos) break;
        a = b + 1;
    }
    return f;
}

bool parse_u32(const std::string& s, uint32_t* v) {
    if (s.empty() || s.size() > 10) return false;
    uint64_t x = 0;
    for (char c : s) {
        if (c < '0' || c > '9') return false;
        x = x * 10 + (uint64_t)(c - '0');
    }
    if (x > 0xFFFFFFFEull) return false;
    *v = (uint32_t)x;
    return true;
}

bool parse_symbol(const std::string& s, unsigned char* c) {
    if (s.size() == 1 && s[0] != '\\') {
        *c = (unsigned char)s[0];
        return true;
    }
    if (s.size() == 4 && s[0] == '\\' && s[1] == 'x') {
        char* e = nullptr;
        const long v = strtol(s.c_str() + 2, &e, 16);
        if (e == s.c_str() + 4 && v >= 0 && v < 256) {
            *c = (unsigned char)v;
            return true;
        }
    }
    return false;
}

int fail(uint32_t line, const char* what) {
    set_error("table text, line %u: %s", line, what);
    return PAREM_EINVAL;
}

}  // namespace

extern "C" int parem_table_write_text(uint32_t num_states, uint32_t alphabet_size, const uint32_t* table,
                                      uint32_t start_state, const uint8_t* accept_bitmap, const char* alphabet,
                                      char* out, size_t cap, size_t* needed) {
    set_error("");
    if (!table || !accept_bitmap || !alphabet || !needed || num_states == 0 || alphabet_size == 0 || alphabet_size > 256 ||
        start_state >= num_states) {
        set_error("table text: bad argument");
        return PAREM_EINVAL;
    }
    std::string o = "symbols";
    for (uint32_t c = 0; c < alphabet_size; ++c) {
        o.push_back('\t');
        put_symbol(o, (unsigned char)alphabet[c]);
    }
    o += "\nstart\t" + std::to_string(start_state) + "\nfinals";
    for (uint32_t s = 0; s < num_states; ++s)
        if (accept_bitmap[s >> 3] >> (s & 7) & 1) o += "\t" + std::to_string(s);
    o.push_back('\n');
    for (uint32_t s = 0; s < num_states; ++s) {
        o += std::to_string(s);
        for (uint32_t c = 0; c < alphabet_size; ++c) {
            const uint32_t d = table[(size_t)s * alphabet_size + c];
            if (d != PAREM_DEAD && d >= num_states) {
                set_error("table text: entry (%u, %u) = %u is neither a state nor DEAD", s, c, d);
                return PAREM_EINVAL;
            }
            o += d == PAREM_DEAD ? std::string("\t-") : "\t" + std::to_string(d);
        }
        o.push_back('\n');
    }
    *needed = o.size();
    if (!out) return PAREM_OK;   // size query
    if (cap < o.size()) {
        set_error("table text: buffer too small: %zu < %zu", cap, o.size());
        return PAREM_ENOMEM;
    }
    memcpy(out, o.data(), o.size());
    return PAREM_OK;
}

extern "C" int parem_table_read_text(const char* text, size_t len, uint32_t max_states, uint32_t* table,
                                     uint8_t* accept_bitmap, parem_regex_info* info) {
    set_error("");
    if (!text || !info) {
        set_error("table text: null argument");
        return PAREM_EINVAL;
    }
    Lines L{text, text + len};
    std::string ln;
    if (!L.next(ln)) return fail(1, "empty text");
    std::vector<std::string> f = split_tabs(ln);
    if (f[0] != "symbols") return fail(L.line, "expected 'symbols<TAB>...'");
    const uint32_t A = (uint32_t)f.size() - 1;
    if (A == 0 || A > 256) return fail(L.line, "1..256 symbols expected");
    memset(info, 0, sizeof(*info));
    bool seen[256] = {false};
    for (uint32_t c = 0; c < A; ++c) {
        unsigned char ch;
        if (!parse_symbol(f[c + 1], &ch)) return fail(L.line, "a symbol is one character or \\xHH");
        if (seen[ch]) return fail(L.line, "duplicate symbol");
        seen[ch] = true;
        info->alphabet[c] = (char)ch;
    }
    if (!L.next(ln)) return fail(L.line + 1, "missing 'start' line");
    f = split_tabs(ln);
    uint32_t start = 0;
    if (f.size() != 2 || f[0] != "start" || !parse_u32(f[1], &start)) return fail(L.line, "expected 'start<TAB><id>'");
    if (!L.next(ln)) return fail(L.line + 1, "missing 'finals' line");
    const uint32_t finals_line = L.line;
    f = split_tabs(ln);
    if (f[0] != "finals") return fail(L.line, "expected 'finals[<TAB><id>...]'");
    std::vector<uint32_t> finals;
    for (size_t i = 1; i < f.size(); ++i) {
        uint32_t v;
        if (!parse_u32(f[i], &v)) return fail(L.line, "bad final state id");
        finals.push_back(v);
    }
    // rows: first pass counts and validates, so a size query needs no output buffers
    std::vector<uint32_t> rows;
    uint32_t Q = 0;
    while (L.next(ln)) {
        if (ln.empty() && L.p >= L.end) break;   // tolerate one trailing empty line
        f = split_tabs(ln);
        uint32_t id;
        if (!parse_u32(f[0], &id) || id != Q) return fail(L.line, "rows must be numbered 0, 1, 2, ... in order");
        if (f.size() != (size_t)A + 1) return fail(L.line, "a row has one entry per symbol");
        for (uint32_t c = 0; c < A; ++c) {
            uint32_t d = PAREM_DEAD;
            if (f[c + 1] != "-" && !parse_u32(f[c + 1], &d)) return fail(L.line, "an entry is a state id or '-'");
            rows.push_back(d);
        }
        ++Q;
    }
    if (Q == 0) return fail(L.line + 1, "no state rows");
    for (size_t i = 0; i < rows.size(); ++i)
        if (rows[i] != PAREM_DEAD && rows[i] >= Q) return fail(4 + (uint32_t)(i / A), "destination out of range");
    if (start >= Q) return fail(2, "start state out of range");
    for (uint32_t v : finals)
        if (v >= Q) return fail(finals_line, "final state out of range");
    info->num_states = Q;
    info->alphabet_size = A;
    info->start_state = start;
    if (!table || !accept_bitmap) return PAREM_OK;   // size query
    if (Q > max_states) {
        set_error("table text: %u states > max_states %u", Q, max_states);
        return PAREM_ENOMEM;
    }
    memcpy(table, rows.data(), rows.size() * sizeof(uint32_t));
    memset(accept_bitmap, 0, (Q + 7) / 8);
    for (uint32_t v : finals) accept_bitmap[v >> 3] |= (uint8_t)(1u << (v & 7));
    return PAREM_OK;
}

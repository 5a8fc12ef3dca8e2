// regex.cpp -- SURVEY §8(f) NEXT-3: the front end of the PaREM tool chain,
// host side.  A regular expression in the paper's language (Table III, P:222-244:
// concatenation, Kleene star, union, positive closure, range [x..y], optionality, groups)
// is parsed into an AST, turned into an NFA by the McNaughton-Yamada-Thompson
// construction (Fig. 5 a-f), made deterministic by the subset construction,
// minimised (Moore partition refinement -- the paper's "optimized" NFA/DFA, made
// canonical) and numbered in breadth-first order from the start state, so the result is
// the unique minimal DFA of the language in a deterministic numbering.  The output is the
// row-major table parem_dfa_create takes.
//
// Alphabet: symbol i is the byte alphabet[i]; with no alphabet given, the distinct bytes
// of the pattern in increasing order.  PAREM_REGEX_SEARCH compiles Sigma* R: the automaton
// of "every occurrence" (the paper's "parallel" automaton, Fig. 1 / Table I, counts every
// position where an occurrence ends).
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <memory>
#include <queue>
#include <string>
#include <vector>

#include "internal.h"

namespace parem {
namespace {

using SymSet = std::vector<bool>;   // over the alphabet

struct Node {
    enum Kind { SYM, CAT, ALT, STAR, PLUS, OPT, EPS } kind;
    SymSet set;                          // SYM
    std::unique_ptr<Node> a, b;
};
using NodeP = std::unique_ptr<Node>;

struct Parser {
    const std::string& s;
    const std::vector<int>& sym_of;   // byte -> symbol id or -1
    uint32_t A;
    size_t i = 0;
    std::string err;

    Parser(const std::string& s_, const std::vector<int>& m, uint32_t a) : s(s_), sym_of(m), A(a) {}

    bool fail(const char* what) {
        if (err.empty()) err = std::string(what) + " at offset " + std::to_string(i);
        return false;
    }
    bool at_end() const { return i >= s.size(); }
    char peek() const { return s[i]; }

    NodeP leaf(SymSet set) {
        NodeP n(new Node{Node::SYM, std::move(set), nullptr, nullptr});
        return n;
    }
    NodeP make(Node::Kind k, NodeP a, NodeP b = nullptr) {
        NodeP n(new Node{k, SymSet(), std::move(a), std::move(b)});
        return n;
    }

    // alt := cat ('|' cat)*
    NodeP alt() {
        NodeP l = cat();
        if (!l) return nullptr;
        while (!at_end() && peek() == '|') {
            ++i;
            NodeP r = cat();
            if (!r) return nullptr;
            l = make(Node::ALT, std::move(l), std::move(r));
        }
        return l;
    }
    // cat := rep* (empty = epsilon)
    NodeP cat() {
        NodeP l;
        while (!at_end() && peek() != '|' && peek() != ')') {
            NodeP r = rep();
            if (!r) return nullptr;
            l = l ? make(Node::CAT, std::move(l), std::move(r)) : std::move(r);
        }
        if (!l) l = make(Node::EPS, nullptr);
        return l;
    }
    // rep := atom ('*' | '+' | '?')*
    NodeP rep() {
        NodeP x = atom();
        if (!x) return nullptr;
        while (!at_end() && (peek() == '*' || peek() == '+' || peek() == '?')) {
            const char op = s[i++];
            x = make(op == '*' ? Node::STAR : op == '+' ? Node::PLUS : Node::OPT, std::move(x));
        }
        return x;
    }
    bool literal(int& sym) {
        if (at_end()) return fail("unexpected end of pattern");
        unsigned char c = (unsigned char)s[i];
        if (c == '\\') {
            ++i;
            if (at_end()) return fail("dangling escape");
            c = (unsigned char)s[i];
        } else if (strchr("()|*+?[]", c)) {
            return fail("unexpected operator");
        }
        ++i;
        sym = sym_of[c];
        if (sym < 0) {
            --i;
            return fail("character not in the alphabet");
        }
        return true;
    }
    NodeP atom() {
        const char c = peek();
        if (c == '(') {
            ++i;
            NodeP x = alt();
            if (!x) return nullptr;
            if (at_end() || peek() != ')') {
                fail("missing ')'");
                return nullptr;
            }
            ++i;
            return x;
        }
        if (c == '[') {   // range [x..y]: every alphabet symbol with x <= byte <= y
            ++i;
            if (i + 5 > s.size() || s[i + 1] != '.' || s[i + 2] != '.' || s[i + 4] != ']') {
                fail("range must read [x..y]");
                return nullptr;
            }
            const unsigned char lo = (unsigned char)s[i], hi = (unsigned char)s[i + 3];
            i += 5;
            if (lo > hi) {
                fail("empty range");
                return nullptr;
            }
            SymSet set(A, false);
            bool any = false;
            for (unsigned v = lo; v <= hi; ++v)
                if (sym_of[v] >= 0) set[sym_of[v]] = any = true;
            if (!any) {
                fail("range matches no alphabet symbol");
                return nullptr;
            }
            return leaf(std::move(set));
        }
        int sym;
        if (!literal(sym)) return nullptr;
        SymSet set(A, false);
        set[sym] = true;
        return leaf(std::move(set));
    }
};

// Thompson NFA: every state has either symbol-set edges or epsilon edges.
struct Nfa {
    struct Edge {
        uint32_t to;
        int set;   // index into sets, -1 = epsilon
    };
    std::vector<std::vector<Edge>> out;
    std::vector<SymSet> sets;
    uint32_t add() {
        out.emplace_back();
        return (uint32_t)out.size() - 1;
    }
    void eps(uint32_t a, uint32_t b) { out[a].push_back({b, -1}); }
    void sym(uint32_t a, uint32_t b, const SymSet& s) {
        sets.push_back(s);
        out[a].push_back({b, (int)sets.size() - 1});
    }
    // McNaughton-Yamada-Thompson, one fragment (start, accept) per AST node (Fig. 5 a-f)
    std::pair<uint32_t, uint32_t> build(const Node& n) {
        const uint32_t s = add(), f = add();
        switch (n.kind) {
            case Node::SYM: sym(s, f, n.set); break;
            case Node::EPS: eps(s, f); break;
            case Node::CAT: {
                auto x = build(*n.a);
                auto y = build(*n.b);
                eps(s, x.first);
                eps(x.second, y.first);
                eps(y.second, f);
                break;
            }
            case Node::ALT: {
                auto x = build(*n.a);
                auto y = build(*n.b);
                eps(s, x.first);
                eps(s, y.first);
                eps(x.second, f);
                eps(y.second, f);
                break;
            }
            case Node::STAR:
            case Node::PLUS:
            case Node::OPT: {
                auto x = build(*n.a);
                eps(s, x.first);
                eps(x.second, f);
                if (n.kind != Node::PLUS) eps(s, f);           // zero occurrences
                if (n.kind != Node::OPT) eps(x.second, x.first);   // repeat
                break;
            }
        }
        return {s, f};
    }
};

void closure(const Nfa& N, std::vector<uint32_t>& set, std::vector<uint32_t>& mark, uint32_t stamp) {
    std::vector<uint32_t> stack(set.begin(), set.end());
    for (uint32_t q : set) mark[q] = stamp;
    while (!stack.empty()) {
        const uint32_t q = stack.back();
        stack.pop_back();
        for (const auto& e : N.out[q])
            if (e.set < 0 && mark[e.to] != stamp) {
                mark[e.to] = stamp;
                set.push_back(e.to);
                stack.push_back(e.to);
            }
    }
    std::sort(set.begin(), set.end());
}

}  // namespace
}  // namespace parem

using namespace parem;

extern "C" int parem_regex_compile(const char* pattern, const char* alphabet, uint32_t flags, uint32_t max_states,
                                   uint32_t* table, uint8_t* accept_bitmap, parem_regex_info* info) {
    set_error("");
    if (!pattern || !info) {
        set_error("null pattern or info");
        return PAREM_EINVAL;
    }
    if (flags & ~PAREM_REGEX_SEARCH) {
        set_error("unknown regex flags 0x%x", flags);
        return PAREM_EINVAL;
    }
    const std::string pat(pattern);
    // ---- alphabet ----
    std::vector<int> sym_of(256, -1);
    std::string alpha;
    if (alphabet && alphabet[0]) {
        alpha = alphabet;
        for (size_t k = 0; k < alpha.size(); ++k) {
            const unsigned char c = (unsigned char)alpha[k];
            if (sym_of[c] >= 0) {
                set_error("alphabet byte 0x%02x repeated", c);
                return PAREM_EINVAL;
            }
            sym_of[c] = (int)k;
        }
    } else {
        std::vector<bool> seen(256, false);
        for (size_t k = 0; k < pat.size(); ++k) {
            unsigned char c = (unsigned char)pat[k];
            if (c == '\\' && k + 1 < pat.size()) {
                seen[(unsigned char)pat[++k]] = true;
                continue;
            }
            if (c == '[' && k + 5 < pat.size() && pat[k + 2] == '.' && pat[k + 3] == '.' && pat[k + 5] == ']') {
                for (unsigned v = (unsigned char)pat[k + 1]; v <= (unsigned char)pat[k + 4]; ++v) seen[v] = true;
                k += 5;
                continue;
            }
            if (!strchr("()|*+?[]", c)) seen[c] = true;
        }
        for (int v = 0; v < 256; ++v)
            if (seen[v]) {
                sym_of[v] = (int)alpha.size();
                alpha.push_back((char)v);
            }
    }
    const uint32_t A = (uint32_t)alpha.size();
    if (A == 0) {
        set_error("empty alphabet");
        return PAREM_EINVAL;
    }
    // ---- AST ----
    Parser ps(pat, sym_of, A);
    NodeP ast = ps.alt();
    if (ast && !ps.at_end()) {
        ps.fail(ps.peek() == ')' ? "unbalanced ')'" : "trailing input");
        ast.reset();
    }
    if (!ast) {
        set_error("regex: %s", ps.err.c_str());
        return PAREM_EINVAL;
    }
    // ---- NFA; SEARCH: a new start with a Sigma self-loop (Sigma* R) ----
    Nfa N;
    auto fr = N.build(*ast);
    uint32_t nstart = fr.first;
    if (flags & PAREM_REGEX_SEARCH) {
        const uint32_t s0 = N.add();
        N.sym(s0, s0, SymSet(A, true));
        N.eps(s0, fr.first);
        nstart = s0;
    }
    const uint32_t nfinal = fr.second;
    // ---- subset construction ----
    const uint32_t cap = max_states ? max_states : 1u << 16;
    std::vector<uint32_t> mark(N.out.size(), 0);
    uint32_t stamp = 0;
    std::map<std::vector<uint32_t>, uint32_t> id;
    std::vector<std::vector<uint32_t>> sets;
    std::vector<uint32_t> dtab;   // [state][A]
    std::vector<uint8_t> dacc;
    std::vector<uint32_t> first{nstart};
    closure(N, first, mark, ++stamp);
    id[first] = 0;
    sets.push_back(first);
    for (size_t q = 0; q < sets.size(); ++q) {
        dacc.push_back(std::binary_search(sets[q].begin(), sets[q].end(), nfinal) ? 1 : 0);
        for (uint32_t c = 0; c < A; ++c) {
            std::vector<uint32_t> nx;
            ++stamp;
            for (uint32_t s : sets[q])
                for (const auto& e : N.out[s])
                    if (e.set >= 0 && N.sets[e.set][c] && mark[e.to] != stamp) {
                        mark[e.to] = stamp;
                        nx.push_back(e.to);
                    }
            closure(N, nx, mark, ++stamp);   // the empty set is the (explicit) dead state
            auto it = id.find(nx);
            uint32_t t;
            if (it == id.end()) {
                t = (uint32_t)sets.size();
                if (t >= 4 * cap + 1024) {
                    set_error("regex: subset construction exceeds %u states (state explosion, P:315)", 4 * cap + 1024);
                    return PAREM_EINVAL;
                }
                id.emplace(nx, t);
                sets.push_back(std::move(nx));
            } else {
                t = it->second;
            }
            dtab.push_back(t);
        }
    }
    const uint32_t n = (uint32_t)sets.size();
    // ---- Moore minimisation: refine {accepting, non-accepting} until stable ----
    std::vector<uint32_t> cls(n), ncls(n);
    for (uint32_t q = 0; q < n; ++q) cls[q] = dacc[q];
    uint32_t ncl = 0;
    for (;;) {
        std::map<std::vector<uint32_t>, uint32_t> sig;
        for (uint32_t q = 0; q < n; ++q) {
            std::vector<uint32_t> key;
            key.reserve(A + 1);
            key.push_back(cls[q]);
            for (uint32_t c = 0; c < A; ++c) key.push_back(cls[dtab[(size_t)q * A + c]]);
            auto it = sig.find(key);
            if (it == sig.end()) it = sig.emplace(std::move(key), (uint32_t)sig.size()).first;
            ncls[q] = it->second;
        }
        const uint32_t k = (uint32_t)sig.size();
        cls.swap(ncls);
        if (k == ncl) break;
        ncl = k;
    }
    // ---- breadth-first numbering from the start class ----
    std::vector<uint32_t> rep(ncl, UINT32_MAX), num(ncl, UINT32_MAX), order;
    for (uint32_t q = 0; q < n; ++q)
        if (rep[cls[q]] == UINT32_MAX) rep[cls[q]] = q;
    std::queue<uint32_t> bfs;
    num[cls[0]] = 0;
    order.push_back(cls[0]);
    bfs.push(cls[0]);
    while (!bfs.empty()) {
        const uint32_t k = bfs.front();
        bfs.pop();
        for (uint32_t c = 0; c < A; ++c) {
            const uint32_t t = cls[dtab[(size_t)rep[k] * A + c]];
            if (num[t] == UINT32_MAX) {
                num[t] = (uint32_t)order.size();
                order.push_back(t);
                bfs.push(t);
            }
        }
    }
    const uint32_t Q = (uint32_t)order.size();
    info->num_states = Q;
    info->alphabet_size = A;
    info->start_state = 0;
    info->reserved = 0;
    memset(info->alphabet, 0, sizeof(info->alphabet));
    memcpy(info->alphabet, alpha.data(), A);
    if (!table || !accept_bitmap) return PAREM_OK;   // size query
    if (Q > cap) {
        set_error("regex: minimal DFA has %u states > max_states %u", Q, cap);
        return PAREM_ENOMEM;
    }
    memset(accept_bitmap, 0, (Q + 7) / 8);
    for (uint32_t j = 0; j < Q; ++j) {
        const uint32_t q = rep[order[j]];
        if (dacc[q]) accept_bitmap[j >> 3] |= (uint8_t)(1u << (j & 7));
        for (uint32_t c = 0; c < A; ++c) table[(size_t)j * A + c] = num[cls[dtab[(size_t)q * A + c]]];
    }
    return PAREM_OK;
}

// Dimension-tree scheduler -- see schedule.hpp for the reference map.
#include "schedule.hpp"

#include <algorithm>
#include <array>
#include <map>

#include "cpdb.h"

namespace cpdb {
namespace {

[[noreturn]] void raise(int code, std::string what) { throw SchedError{code, std::move(what)}; }

std::string set_name(ModeSet s, uint32_t order) {
    std::string out = "Y(";
    bool first = true;
    for (uint32_t m = 0; m < order; ++m)
        if (s & (1u << m)) {
            if (!first) out += ',';
            out += std::to_string(m + 1);
            first = false;
        }
    return out + ")";
}

// Plan text: updates separated by '|', "<mode>:<step>,<step>..." with a step
// written "<source>.<contracted mode>", source "X" for the root or the digits of
// its free modes (0-based).  Same data as dim_tree.hpp:240-310.
Sweep parse(const char* text, uint32_t order) {
    Sweep sw;
    const ModeSet root = (1u << order) - 1u;
    const char* p = text;
    while (*p) {
        Update u;
        u.mode = static_cast<uint32_t>(*p - '0');
        p += 2;  // digit + ':'
        while (*p && *p != '|') {
            ModeSet src = 0;
            if (*p == 'X') {
                src = root;
                ++p;
            } else {
                while (*p != '.') src |= 1u << (*p++ - '0');
            }
            ++p;  // '.'
            const uint32_t c = static_cast<uint32_t>(*p++ - '0');
            u.steps.push_back({src, c, src & ~(1u << c)});
            if (*p == ',') ++p;
        }
        if (*p == '|') ++p;
        sw.updates.push_back(std::move(u));
    }
    return sw;
}

constexpr const char* kTree3 = "0:X.2,01.1|1:01.0|2:X.1,02.0";
constexpr const char* kTree4 = "0:X.3,012.2,01.1|1:01.0|2:012.1,02.0|3:X.0,123.1,23.2";
constexpr const char* kReuse3Even = "0:02.2|2:02.0|1:X.0,12.2";
constexpr const char* kReuse3Odd = "1:12.2|2:12.1|0:X.1,02.2";
constexpr const char* kReuse4Second = "2:23.3|3:23.2|1:123.2,13.3|0:X.1,023.2,03.3";
constexpr const char* kReuse4Third = "0:03.3|2:023.3,02.0|3:023.2,03.0|1:X.2,013.0,13.3";

// Naive inner orders (dim_tree.hpp:210-224)
Sweep naive_sweep(uint32_t order) {
    static const uint32_t t3[3][2] = {{2, 1}, {0, 2}, {1, 0}};
    static const uint32_t t4[4][3] = {{3, 2, 1}, {3, 2, 0}, {0, 1, 3}, {0, 1, 2}};
    Sweep sw;
    for (uint32_t mode = 0; mode < order; ++mode) {
        std::vector<uint32_t> seq;
        if (order == 3) seq.assign(t3[mode], t3[mode] + 2);
        else if (order == 4) seq.assign(t4[mode], t4[mode] + 3);
        else
            for (uint32_t k = order; k-- > 0;)
                if (k != mode) seq.push_back(k);
        Update u{mode, {}};
        ModeSet cur = (1u << order) - 1u;
        for (uint32_t c : seq) {
            u.steps.push_back({cur, c, cur & ~(1u << c)});
            cur &= ~(1u << c);
        }
        sw.updates.push_back(std::move(u));
    }
    return sw;
}

ModeSet permute(ModeSet s, const std::array<uint32_t, 4>& perm) {
    ModeSet out = 0;
    for (uint32_t m = 0; m < 4; ++m)
        if (s & (1u << m)) out |= 1u << perm[m];
    return out;
}

Sweep permute(const Sweep& in, const std::array<uint32_t, 4>& perm) {
    Sweep out;
    for (const auto& u : in.updates) {
        Update v{perm[u.mode], {}};
        for (const auto& st : u.steps)
            v.steps.push_back({permute(st.source, perm), perm[st.contract],
                               permute(st.produces, perm)});
        out.updates.push_back(std::move(v));
    }
    return out;
}

bool same_structure(const Sweep& a, const Sweep& b) {
    if (a.updates.size() != b.updates.size()) return false;
    for (size_t i = 0; i < a.updates.size(); ++i) {
        const auto& u = a.updates[i];
        const auto& v = b.updates[i];
        if (u.mode != v.mode || u.steps.size() != v.steps.size()) return false;
        for (size_t k = 0; k < u.steps.size(); ++k)
            if (u.steps[k].source != v.steps[k].source || u.steps[k].contract != v.steps[k].contract)
                return false;
    }
    return true;
}

}  // namespace

std::vector<uint32_t> Plan::update_order(uint64_t i) const {
    std::vector<uint32_t> o;
    for (const auto& u : sweeps.at(i).updates) o.push_back(u.mode);
    return o;
}

uint64_t Plan::pattern_of(uint64_t i) const {
    for (uint64_t j = 0; j < i; ++j)
        if (same_structure(sweeps[j], sweeps[i])) return j;
    return i;
}

Plan build_plan(uint32_t order, Strategy strategy, uint64_t n) {
    if (n == 0) raise(CPDB_INVALID_ARGUMENT, "build_schedule: need at least one iteration");
    if (order < 2) raise(CPDB_INVALID_ARGUMENT, "build_schedule: order must be >= 2");
    if (strategy != Strategy::naive && order != 3 && order != 4)
        raise(CPDB_INVALID_ARGUMENT,
              "build_schedule: tree strategies are defined for orders 3 and 4 only");
    if (order >= 32) raise(CPDB_INVALID_ARGUMENT, "build_schedule: order too large");
    Plan p;
    p.order = order;
    p.strategy = strategy;
    p.sweeps.reserve(n);
    switch (strategy) {
        case Strategy::naive:
            p.sweeps.assign(n, naive_sweep(order));
            break;
        case Strategy::dim_tree:
            p.sweeps.assign(n, parse(order == 3 ? kTree3 : kTree4, order));
            break;
        case Strategy::branch_reuse:
            if (order == 3) {
                // 2-cycle from sweep 2 (dim_tree.hpp:404-410)
                p.cycle_start = 1;
                p.cycle_length = 2;
                const Sweep cyc[2] = {parse(kReuse3Even, 3), parse(kReuse3Odd, 3)};
                p.sweeps.push_back(parse(kTree3, 3));
                for (uint64_t i = 1; i < n; ++i) p.sweeps.push_back(cyc[(i - 1) % 2]);
            } else {
                // sigma = (1,2,0,3) rotation of the third pattern (dim_tree.hpp:411-422)
                p.cycle_start = 2;
                p.cycle_length = 3;
                static const std::array<uint32_t, 4> sigma = {1, 2, 0, 3};
                p.sweeps.push_back(parse(kTree4, 4));
                if (n > 1) p.sweeps.push_back(parse(kReuse4Second, 4));
                if (n > 2) p.sweeps.push_back(parse(kReuse4Third, 4));
                for (uint64_t i = 3; i < n; ++i) p.sweeps.push_back(permute(p.sweeps[i - 1], sigma));
            }
            break;
        default:
            raise(CPDB_INVALID_ARGUMENT, "build_schedule: unknown strategy");
    }
    validate_plan(p);
    return p;
}

void validate_plan(const Plan& p) {
    const uint32_t order = p.order;
    const ModeSet root = p.root();
    std::vector<uint64_t> version(order, 1);
    std::map<ModeSet, std::vector<uint64_t>> stamps;  // 0 = not absorbed
    for (uint64_t i = 0; i < p.sweeps.size(); ++i) {
        const auto& sw = p.sweeps[i];
        if (sw.updates.size() != order)
            raise(CPDB_LOGIC_ERROR, "schedule: iteration must update every mode exactly once");
        ModeSet seen = 0;
        for (const auto& u : sw.updates) {
            if (u.mode >= order || (seen & (1u << u.mode)))
                raise(CPDB_LOGIC_ERROR, "schedule: duplicate or out-of-range update mode");
            seen |= 1u << u.mode;
            if (u.steps.empty() || u.steps.back().produces != (1u << u.mode))
                raise(CPDB_LOGIC_ERROR, "schedule: update must end in its final tensor");
            for (const auto& s : u.steps) {
                if (s.contract >= order || !(s.source & (1u << s.contract)))
                    raise(CPDB_LOGIC_ERROR, "schedule: contract mode not free in source");
                if (s.produces != (s.source & ~(1u << s.contract)))
                    raise(CPDB_LOGIC_ERROR, "schedule: produced set must drop the contracted mode");
                std::vector<uint64_t> cur(order, 0);
                if (s.source != root) {
                    auto it = stamps.find(s.source);
                    if (it == stamps.end())
                        raise(CPDB_LOGIC_ERROR, "schedule: source " + set_name(s.source, order) +
                                                    " not available at iteration " +
                                                    std::to_string(i + 1));
                    for (uint32_t m = 0; m < order; ++m)
                        if (it->second[m] && it->second[m] != version[m])
                            raise(CPDB_STALE_INTERMEDIATE,
                                  "schedule: stale source " + set_name(s.source, order) +
                                      " at iteration " + std::to_string(i + 1) +
                                      ", update of mode " + std::to_string(u.mode + 1));
                    cur = it->second;
                }
                cur[s.contract] = version[s.contract];
                if (s.produces != (1u << u.mode)) stamps[s.produces] = cur;
            }
            ++version[u.mode];
        }
    }
}

std::vector<ModeSet> retained_keys(const Plan& p, uint64_t sweep, uint32_t block) {
    uint64_t next = sweep + 1;
    const uint64_t n = p.sweeps.size();
    if (next >= n) {
        if (next > p.cycle_start) next = p.cycle_start + (next - p.cycle_start) % p.cycle_length;
        if (next >= n) next = n - 1;
    }
    const Sweep* horizon[2] = {&p.sweeps.at(sweep), &p.sweeps.at(next)};
    std::vector<ModeSet> needed, written;
    const ModeSet root = p.root();
    for (int h = 0; h < 2; ++h)
        for (uint32_t b = 0; b < horizon[h]->updates.size(); ++b) {
            if (h == 0 && b <= block) continue;
            for (const auto& s : horizon[h]->updates[b].steps) {
                if (s.source != root &&
                    std::find(written.begin(), written.end(), s.source) == written.end())
                    needed.push_back(s.source);
                written.push_back(s.produces);
            }
        }
    return needed;
}

Cost measured_cost(const Plan& p, const std::vector<uint64_t>& dims, uint64_t rank,
                   uint64_t sweeps) {
    if (dims.size() != p.order)
        raise(CPDB_INVALID_ARGUMENT, "measured_cost: dims do not match schedule order");
    Cost c;
    const ModeSet root = p.root();
    for (uint64_t i = 0; i < sweeps && i < p.sweeps.size(); ++i)
        for (const auto& u : p.sweeps[i].updates)
            for (const auto& s : u.steps) {
                uint64_t f = 2;
                for (uint32_t m = 0; m < p.order; ++m)
                    if (s.source & (1u << m)) f *= dims[m];
                const uint32_t rpow = p.order - popcount(s.source) + 1;
                for (uint32_t k = 0; k < rpow; ++k) f *= rank;
                c.flops += f;
                if (s.source == root) ++c.roots;
            }
    return c;
}

uint64_t closed_form_cost(uint32_t order, Strategy s, const std::vector<uint64_t>& d,
                          uint64_t R) {
    if (order != 3 && order != 4)
        raise(CPDB_INVALID_ARGUMENT, "closed_form_cost: order must be 3 or 4");
    if (d.size() != order) raise(CPDB_INVALID_ARGUMENT, "closed_form_cost: dims do not match order");
    // Sum of coefficient * prod(extents of set) * R^power; tables restate
    // dim_tree.hpp:593-619 as (coeff, set bitmask, power) triples.
    struct Term {
        uint64_t coeff;
        ModeSet set;
        uint32_t pow;
    };
    static const std::vector<Term> t3[3] = {
        {{18, 0x7, 1}, {6, 0x3, 2}, {6, 0x6, 2}, {6, 0x5, 2}},
        {{12, 0x7, 1}, {12, 0x3, 2}, {6, 0x5, 2}},
        {{8, 0x7, 1}, {4, 0x3, 2}, {8, 0x5, 2}, {6, 0x6, 2}}};
    static const std::vector<Term> t4[3] = {
        {{24, 0xF, 1}, {12, 0x7, 2}, {12, 0xE, 2}, {12, 0x3, 3}, {12, 0xC, 3}},
        {{12, 0xF, 1}, {12, 0x7, 2}, {6, 0xE, 2}, {12, 0x3, 3}, {6, 0x5, 3}, {6, 0xC, 3}},
        {{8, 0xF, 1}, {4, 0x7, 2}, {4, 0xE, 2}, {6, 0xD, 2}, {2, 0xB, 2}, {4, 0x3, 3},
         {4, 0x5, 3}, {6, 0xC, 3}, {6, 0x9, 3}, {4, 0xA, 3}}};
    const auto& terms = (order == 3 ? t3 : t4)[static_cast<int>(s)];
    uint64_t total = 0;
    for (const auto& t : terms) {
        uint64_t v = t.coeff;
        for (uint32_t m = 0; m < order; ++m)
            if (t.set & (1u << m)) v *= d[m];
        for (uint32_t k = 0; k < t.pow; ++k) v *= R;
        total += v;
    }
    return total;
}

uint64_t leading_flop_coefficient(uint32_t order, Strategy s) {
    if (order != 3 && order != 4)
        raise(CPDB_INVALID_ARGUMENT, "leading_flop_coefficient: order must be 3 or 4");
    switch (s) {
        case Strategy::naive: return order == 3 ? 18 : 24;
        case Strategy::dim_tree: return 12;
        case Strategy::branch_reuse: return 8;
    }
    raise(CPDB_INVALID_ARGUMENT, "leading_flop_coefficient: unknown strategy");
}

}  // namespace cpdb

// Happens-before checker for the multi-stream sweep (diagnostic, CPDB_HBCHECK=1).
//
// The session issues its kernels on up to seven streams whose ordering is
// expressed only through events.  A missing event shows up as a
// timing-dependent result (a kernel reads a buffer its producer has not
// finished, or overwrites one a consumer still reads).  This checker replays
// the issue order on the host with vector clocks -- one clock per stream,
// events capture the recording stream's clock, a wait joins it, a host
// synchronisation joins the host's clock into every later issue -- and
// checks every declared buffer access against the last write and the reads
// since (the FastTrack rule).  Violations are reported deterministically,
// independent of how the GPU happened to schedule the run.
//
// Same-stream order counts as a full dependency: every hot-path kernel that
// is launched programmatically starts with griddepcontrol.wait (pdl_entry,
// device.cuh), which returns once the previous grid has completed and its
// writes are visible.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

namespace cpdb {

struct HbCheck {
    struct Acc {
        int sid = -1;
        uint64_t tick = 0;
        const char* what = "";
        uint64_t sweep = 0;
        uint32_t mode = 0;
    };
    struct Entry {
        uintptr_t lo, hi;
        Acc w;
        std::vector<Acc> r;
    };
    struct Rg {
        const void* p;
        size_t bytes;
    };
    using VC = std::vector<uint64_t>;

    bool on = false;
    uint64_t cur_sweep = 0;  // tags of the next ops (set by the issuer)
    uint32_t cur_mode = 0;
    uint64_t violations = 0;
    std::map<cudaStream_t, int> sid;
    std::vector<VC> vc;  // per stream
    std::map<cudaEvent_t, VC> ev;
    VC host;
    std::vector<Entry> mem;
    std::vector<std::string> names;

    int id(cudaStream_t s) {
        auto it = sid.find(s);
        if (it != sid.end()) return it->second;
        const int n = int(vc.size());
        sid[s] = n;
        vc.emplace_back();
        names.push_back("stream" + std::to_string(n));
        return n;
    }
    void name(cudaStream_t s, const char* nm) { names[id(s)] = nm; }
    static void join(VC& a, const VC& b) {
        if (a.size() < b.size()) a.resize(b.size(), 0);
        for (size_t i = 0; i < b.size(); ++i)
            if (b[i] > a[i]) a[i] = b[i];
    }
    bool before(const Acc& a, int s) const {
        if (a.sid < 0) return true;
        const VC& v = vc[s];
        return size_t(a.sid) < v.size() && v[a.sid] >= a.tick;
    }
    void record(cudaEvent_t e, cudaStream_t s) {
        if (!on) return;
        const int i = id(s);
        join(vc[i], host);
        ev[e] = vc[i];
    }
    void wait(cudaStream_t s, cudaEvent_t e) {
        if (!on) return;
        const int i = id(s);
        auto it = ev.find(e);
        if (it != ev.end()) join(vc[i], it->second);
    }
    void sync_stream(cudaStream_t s) {
        if (on) join(host, vc[id(s)]);
    }
    void sync_event(cudaEvent_t e) {
        if (!on) return;
        auto it = ev.find(e);
        if (it != ev.end()) join(host, it->second);
    }
    void sync_all() {
        if (!on) return;
        for (const VC& v : vc) join(host, v);
    }
    void report(const char* kind, const char* what, int s, const Acc& other, const Rg& g) {
        ++violations;
        const VC& v = vc[s];
        if (violations <= 40)
            std::fprintf(stderr,
                         "cpdb hbcheck: %s race: %s on %s (sweep %llu mode %u) vs %s on %s (sweep "
                         "%llu mode %u, tick %llu; %s has seen tick %llu), buffer %p +%zu\n",
                         kind, what, names[s].c_str(), (unsigned long long)cur_sweep, cur_mode,
                         other.what, names[other.sid].c_str(), (unsigned long long)other.sweep,
                         other.mode, (unsigned long long)other.tick, names[s].c_str(),
                         (unsigned long long)(size_t(other.sid) < v.size() ? v[other.sid] : 0),
                         g.p, g.bytes);
    }
    // One operation on stream s reading `rd` and writing `wr`.
    void op(cudaStream_t s, const char* what, std::initializer_list<Rg> rd,
            std::initializer_list<Rg> wr) {
        if (!on) return;
        const int i = id(s);
        join(vc[i], host);
        if (vc[i].size() <= size_t(i)) vc[i].resize(i + 1, 0);
        const Acc me{i, ++vc[i][i], what, cur_sweep, cur_mode};
        for (const Rg& g : rd) {
            if (!g.p || !g.bytes) continue;
            const uintptr_t lo = uintptr_t(g.p), hi = lo + g.bytes;
            bool exact = false;
            for (Entry& e : mem) {
                if (e.hi <= lo || e.lo >= hi) continue;
                if (!before(e.w, i)) report("read-after-write", what, i, e.w, g);
                if (e.lo == lo && e.hi == hi) {
                    e.r.push_back(me);
                    exact = true;
                }
            }
            if (!exact) mem.push_back(Entry{lo, hi, Acc{}, {me}});
        }
        for (const Rg& g : wr) {
            if (!g.p || !g.bytes) continue;
            const uintptr_t lo = uintptr_t(g.p), hi = lo + g.bytes;
            for (Entry& e : mem) {
                if (e.hi <= lo || e.lo >= hi) continue;
                if (!before(e.w, i)) report("write-after-write", what, i, e.w, g);
                for (const Acc& r : e.r)
                    if (r.sid != i && !before(r, i)) report("write-after-read", what, i, r, g);
            }
            std::vector<Entry> keep;
            for (Entry& e : mem)
                if (!(e.lo >= lo && e.hi <= hi)) keep.push_back(std::move(e));
            keep.push_back(Entry{lo, hi, me, {}});
            mem.swap(keep);
        }
    }
};

}  // namespace cpdb

// planner.cpp -- ADHA host planner: ODS and PDL.
//
// ODS, "optimal data-layout of a section": an affinity graph
// over the section's fields whose edge weight counts common occurrences
// (trip*freq weighted, reading Q11), then greedy
// clustering bounded by an architecture cluster size (Kruskal
// with inclusive byte capacity and tie-break (weight desc, min decl, max decl),
// SPEC.md:133, readings Q13/Q14).  Fields the section does not touch stay
// singletons.
//
// PDL, "program data-layout": combine edges are realised as
// runs of contiguous sections sharing the ODS layout of their merge (PAPER.md:
// 53-54), remap edges cost moved bytes / bandwidth + overhead
// (reading Q19), execution times come from the
// tuning profile when present else the analytic model of
// SPEC.md:205-207, and the plan is the shortest path (ties per
// SPEC.md:283).
#include <algorithm>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "internal.h"
#include "json.h"

namespace adha {
namespace planner {

struct PlanError : std::runtime_error {
    adha_status code;
    PlanError(adha_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Group {
    std::vector<int> fields;     // decl indices
    std::vector<char> in;        // membership by decl index
    double freq = 1.0;
    bool streaming = false;
    double ops = 0.0;
};

struct Section {
    std::string id;
    double trip = 1.0;
    std::vector<Group> groups;
    std::vector<std::string> allowed;
    std::vector<char> touched;   // union of group fields, by decl index
};

struct Device {
    std::string name;
    double line_bytes = 64, line_time = 1, throughput = 1, penalty = 2;
    bool coalescing = false;
    double capacity = 64;
};

struct Link {
    std::string a, b;
    double bw = 1, lat = 0;
};

struct Program {
    int64_t record_count = 0;
    std::vector<std::string> names;
    std::vector<double> eb;
    std::vector<Section> sections;
    std::vector<int> order;      // indices into sections
};

struct Arch {
    std::vector<Device> devices;
    std::vector<Link> links;
    double same_bw = 1, overhead = 0;
    const Device& dev(const std::string& n) const {
        for (auto& d : devices)
            if (d.name == n) return d;
        throw PlanError(ADHA_ERR_PLANNER, "unknown device '" + n + "'");
    }
};

using PLayout = std::vector<std::vector<int>>;  // canonical clusters of decl indices
using Profile = std::map<std::string, double>;  // key: section \x1f device \x1f layout

// ----------------------------------------------------------------------------- parsing

static Program parse_program(const std::string& text) {
    json::Value v = json::parse(text);
    Program p;
    p.record_count = (int64_t)v.at("record_count").as_num();
    std::map<std::string, int> idx;
    for (auto& f : v.at("fields").as_arr()) {
        const std::string& n = f.at("name").as_str();
        if (!idx.emplace(n, (int)p.names.size()).second)
            throw PlanError(ADHA_ERR_PLANNER, "duplicate field '" + n + "'");
        p.names.push_back(n);
        double eb = f.at("elem_bytes").as_num();
        if (!(eb >= 1)) throw PlanError(ADHA_ERR_PLANNER, "field '" + n + "' has elem_bytes < 1");
        p.eb.push_back(eb);
    }
    const int F = (int)p.names.size();
    std::map<std::string, int> sidx;
    for (auto& s : v.at("sections").as_arr()) {
        Section S;
        S.id = s.at("id").as_str();
        S.trip = s.at("trip_count").as_num();
        S.touched.assign(F, 0);
        for (auto& d : s.at("allowed_devices").as_arr()) S.allowed.push_back(d.as_str());
        for (auto& g : s.at("groups").as_arr()) {
            Group G;
            G.in.assign(F, 0);
            for (auto& fn : g.at("fields").as_arr()) {
                auto it = idx.find(fn.as_str());
                if (it == idx.end())
                    throw PlanError(ADHA_ERR_PLANNER, "section '" + S.id + "' uses undeclared field '" +
                                                          fn.as_str() + "'");
                if (!G.in[it->second]) G.fields.push_back(it->second);
                G.in[it->second] = 1;
                S.touched[it->second] = 1;
            }
            G.freq = g.at("freq").as_num();
            const std::string& pat = g.at("pattern").as_str();
            if (pat == "streaming") G.streaming = true;
            else if (pat == "irregular") G.streaming = false;
            else throw PlanError(ADHA_ERR_PLANNER, "bad pattern '" + pat + "'");
            if (const json::Value* o = g.find("ops")) G.ops = o->as_num();
            S.groups.push_back(std::move(G));
        }
        if (!sidx.emplace(S.id, (int)p.sections.size()).second)
            throw PlanError(ADHA_ERR_PLANNER, "duplicate section '" + S.id + "'");
        p.sections.push_back(std::move(S));
    }
    if (const json::Value* o = v.find("order")) {
        for (auto& s : o->as_arr()) {
            auto it = sidx.find(s.as_str());
            if (it == sidx.end()) throw PlanError(ADHA_ERR_PLANNER, "order names unknown section '" + s.as_str() + "'");
            p.order.push_back(it->second);
        }
    } else {
        for (int i = 0; i < (int)p.sections.size(); ++i) p.order.push_back(i);
    }
    return p;
}

static Arch parse_arch(const std::string& text) {
    json::Value v = json::parse(text);
    Arch a;
    for (auto& d : v.at("devices").as_arr()) {
        Device D;
        D.name = d.at("name").as_str();
        D.line_bytes = d.at("line_bytes").as_num();
        D.line_time = d.at("line_time_ns").as_num();
        D.throughput = d.at("throughput_ops_per_ns").as_num();
        D.coalescing = d.at("coalescing").as_bool();
        D.penalty = d.has("stream_cluster_penalty") ? d.at("stream_cluster_penalty").as_num() : 2.0;
        D.capacity = d.at("cluster_capacity_bytes").as_num();
        a.devices.push_back(D);
    }
    if (const json::Value* l = v.find("links")) {
        for (auto& x : l->as_arr())
            a.links.push_back({x.at("from").as_str(), x.at("to").as_str(),
                               x.at("bandwidth_bytes_per_ns").as_num(), x.at("latency_ns").as_num()});
    }
    a.same_bw = v.at("same_device_remap_bandwidth_bytes_per_ns").as_num();
    a.overhead = v.at("remap_fixed_overhead_ns").as_num();
    return a;
}

static std::string pkey(const std::string& s, const std::string& d, const std::string& l) {
    return s + '\x1f' + d + '\x1f' + l;
}

static Profile parse_profile(const char* text) {
    Profile pr;
    if (!text) return pr;
    json::Value v = json::parse(text);
    const json::Value* entries = &v;
    if (v.kind == json::Value::Object) entries = &v.at("entries");
    for (auto& e : entries->as_arr())
        pr[pkey(e.at("section").as_str(), e.at("device").as_str(), e.at("layout").as_str())] =
            e.at("time_ns").as_num();
    return pr;
}

// ----------------------------------------------------------------------------- layouts

static PLayout canonical(PLayout l) {
    for (auto& c : l) std::sort(c.begin(), c.end());
    l.erase(std::remove_if(l.begin(), l.end(), [](const std::vector<int>& c) { return c.empty(); }), l.end());
    std::sort(l.begin(), l.end(), [](const std::vector<int>& a, const std::vector<int>& b) { return a[0] < b[0]; });
    return l;
}

static std::string lstring(const Program& p, const PLayout& l) {
    std::string s;
    for (size_t c = 0; c < l.size(); ++c) {
        if (c) s += '|';
        s += '{';
        for (size_t k = 0; k < l[c].size(); ++k) {
            if (k) s += ',';
            s += p.names[l[c][k]];
        }
        s += '}';
    }
    return s;
}

static double cbytes(const Program& p, const std::vector<int>& c) {
    double b = 0;
    for (int f : c) b += p.eb[f];
    return b;
}

// ----------------------------------------------------------------------------- ODS

static bool allowed(const Section& s, const std::string& d) {
    return std::find(s.allowed.begin(), s.allowed.end(), d) != s.allowed.end();
}

static PLayout ods(const Section& s, const Device& d, const Program& p) {
    if (!allowed(s, d.name))
        throw PlanError(ADHA_ERR_PLANNER, "device '" + d.name + "' not allowed for section '" + s.id + "'");
    const int F = (int)p.names.size();
    std::vector<int> nodes;
    for (int f = 0; f < F; ++f)
        if (s.touched[f]) nodes.push_back(f);
    for (int f : nodes)
        if (p.eb[f] > d.capacity)
            throw PlanError(ADHA_ERR_CAPACITY, "field '" + p.names[f] + "' wider than the cluster capacity of '" +
                                                   d.name + "'");
    // affinity graph: weight(f,g) = sum over groups containing both of trip*freq*w_d
    std::map<std::pair<int, int>, double> w;
    for (const Group& g : s.groups) {
        const double wd = g.streaming ? (d.coalescing ? -1.0 : 1.0) : 1.0;
        std::vector<int> mem = g.fields;
        std::sort(mem.begin(), mem.end());
        for (size_t i = 0; i < mem.size(); ++i)
            for (size_t j = i + 1; j < mem.size(); ++j) {
                auto& slot = w[{mem[i], mem[j]}];
                slot += s.trip * g.freq * wd;
            }
    }
    struct Edge { double w; int a, b; };
    std::vector<Edge> edges;
    edges.reserve(w.size());
    for (auto& kv : w) edges.push_back({kv.second, kv.first.first, kv.first.second});
    std::sort(edges.begin(), edges.end(), [](const Edge& x, const Edge& y) {
        if (x.w != y.w) return x.w > y.w;
        if (x.a != y.a) return x.a < y.a;
        return x.b < y.b;
    });
    // Kruskal greedy with a byte capacity (inclusive)
    std::vector<int> parent(F);
    std::vector<double> bytes(F);
    for (int f = 0; f < F; ++f) { parent[f] = f; bytes[f] = p.eb[f]; }
    auto find = [&](int x) {
        while (parent[x] != x) x = parent[x] = parent[parent[x]];
        return x;
    };
    for (const Edge& e : edges) {
        if (!(e.w > 0)) continue;
        int ra = find(e.a), rb = find(e.b);
        if (ra == rb) continue;
        if (bytes[ra] + bytes[rb] > d.capacity) continue;
        parent[rb] = ra;
        bytes[ra] += bytes[rb];
    }
    std::map<int, std::vector<int>> groups;
    for (int f = 0; f < F; ++f) groups[s.touched[f] ? find(f) : -1 - f].push_back(f);
    PLayout l;
    for (auto& kv : groups) l.push_back(kv.second);
    return canonical(l);
}

static Section merge(const Program& p, const std::vector<int>& secs) {
    Section m;
    m.trip = 1.0;
    m.touched.assign(p.names.size(), 0);
    for (size_t k = 0; k < secs.size(); ++k) {
        const Section& s = p.sections[secs[k]];
        m.id += (k ? "+" : "") + s.id;
        for (const Group& g : s.groups) {
            Group h = g;
            h.freq = s.trip * g.freq;
            m.groups.push_back(h);
        }
        for (size_t f = 0; f < s.touched.size(); ++f) m.touched[f] |= s.touched[f];
    }
    for (const std::string& d : p.sections[secs[0]].allowed) {
        bool all = true;
        for (size_t k = 1; k < secs.size(); ++k) all = all && allowed(p.sections[secs[k]], d);
        if (all) m.allowed.push_back(d);
    }
    if (m.allowed.empty()) throw PlanError(ADHA_ERR_PLANNER, "merged sections share no device");
    return m;
}

// ----------------------------------------------------------------------------- costs

static double exec_cost(const Section& s, const PLayout& l, const Device& d, const Program& p,
                        const Profile& prof) {
    if (!prof.empty()) {
        auto it = prof.find(pkey(s.id, d.name, lstring(p, l)));
        if (it != prof.end()) return it->second;
    }
    double memory = 0.0, compute = 0.0;
    for (const Group& g : s.groups) {
        double inner = 0.0;
        for (const auto& c : l) {
            bool touch = false;
            for (int f : c) touch = touch || g.in[f];
            if (!touch) continue;
            double lc;
            if (g.streaming) {
                lc = cbytes(p, c) / d.line_bytes;
                if (d.coalescing && c.size() > 1) lc = lc * d.penalty;
            } else {
                lc = 1.0;
            }
            inner += lc * d.line_time;
        }
        memory += s.trip * g.freq * inner;
        compute += s.trip * g.freq * g.ops / d.throughput;
    }
    return memory + compute;
}

static std::vector<int> cluster_members(const PLayout& l, int f) {
    for (auto& c : l)
        if (std::find(c.begin(), c.end(), f) != c.end()) return c;
    return {};
}

// moved fields sorted by name
static std::vector<int> moved_fields(const Program& p, const PLayout& l1, const std::string& d1,
                                     const PLayout& l2, const std::string& d2, const std::vector<char>& common) {
    std::vector<int> moved;
    const int F = (int)p.names.size();
    for (int f = 0; f < F; ++f) {
        if (!common[f]) continue;
        if (d1 != d2) { moved.push_back(f); continue; }
        std::vector<int> a, b;
        for (int x : cluster_members(l1, f)) if (common[x]) a.push_back(x);
        for (int x : cluster_members(l2, f)) if (common[x]) b.push_back(x);
        std::sort(a.begin(), a.end());
        std::sort(b.begin(), b.end());
        if (a != b) moved.push_back(f);
    }
    std::sort(moved.begin(), moved.end(), [&](int x, int y) { return p.names[x] < p.names[y]; });
    return moved;
}

static double remap_cost(const Program& p, const Arch& a, const PLayout& l1, const std::string& d1,
                         const PLayout& l2, const std::string& d2, const std::vector<char>& common,
                         std::vector<int>* moved_out) {
    std::vector<int> moved = moved_fields(p, l1, d1, l2, d2, common);
    double nbytes = 0.0;
    for (int f : moved) nbytes += (double)p.record_count * p.eb[f];
    if (moved_out) *moved_out = moved;
    if (nbytes == 0) return 0.0;
    if (d1 == d2) return nbytes / a.same_bw + a.overhead;
    for (const Link& lk : a.links)
        if ((lk.a == d1 && lk.b == d2) || (lk.a == d2 && lk.b == d1)) return nbytes / lk.bw + lk.lat;
    throw PlanError(ADHA_ERR_PLANNER, "no link between '" + d1 + "' and '" + d2 + "'");
}

// ----------------------------------------------------------------------------- PDL

struct Run {
    int begin, end;
    std::string device;
    PLayout layout;
    double exec_ns;
    std::vector<char> fields;
};

static Run make_run(const Program& p, const Arch& a, int b, int e, const Device& d, const Profile& prof) {
    std::vector<int> secs(p.order.begin() + b, p.order.begin() + e + 1);
    Run r{b, e, d.name, ods(merge(p, secs), d, p), 0.0, std::vector<char>(p.names.size(), 0)};
    for (int si : secs) {
        const Section& s = p.sections[si];
        r.exec_ns += exec_cost(s, r.layout, d, p, prof);
        for (size_t f = 0; f < s.touched.size(); ++f) r.fields[f] |= s.touched[f];
    }
    return r;
}

static std::vector<char> intersect(const std::vector<char>& x, const std::vector<char>& y) {
    std::vector<char> z(x.size());
    for (size_t i = 0; i < x.size(); ++i) z[i] = x[i] && y[i];
    return z;
}

struct Path {
    double cost;
    std::vector<int> nodes;
};

// (cost, n_runs, [(device, begin) ...]) lexicographic
static bool path_less(const std::vector<Run>& R, const Path& x, const Path& y) {
    if (x.cost != y.cost) return x.cost < y.cost;
    if (x.nodes.size() != y.nodes.size()) return x.nodes.size() < y.nodes.size();
    for (size_t i = 0; i < x.nodes.size(); ++i) {
        const Run& a = R[x.nodes[i]];
        const Run& b = R[y.nodes[i]];
        if (a.device != b.device) return a.device < b.device;
        if (a.begin != b.begin) return a.begin < b.begin;
    }
    return false;
}

// the run graph's nodes: every contiguous run x every device allowed by all members
static std::vector<Run> run_nodes(const Program& p, const Arch& a, const Profile& prof) {
    const int k = (int)p.order.size();
    if (k == 0) throw PlanError(ADHA_ERR_PLANNER, "program has no sections");
    for (auto& s : p.sections)
        for (auto& d : s.allowed) a.dev(d);   // validate device names
    std::vector<Run> R;
    for (int b = 0; b < k; ++b)
        for (int e = b; e < k; ++e)
            for (const Device& d : a.devices) {
                bool ok = true;
                for (int i = b; i <= e; ++i) ok = ok && allowed(p.sections[p.order[i]], d.name);
                if (ok) R.push_back(make_run(p, a, b, e, d, prof));
            }
    return R;
}

static std::string candidates_json(const Program& p, const Arch& a, const Profile& prof) {
    std::vector<Run> R = run_nodes(p, a, prof);
    std::string out = "{\"schema_version\":1,\"runs\":[";
    for (size_t r = 0; r < R.size(); ++r) {
        const Run& x = R[r];
        if (r) out += ',';
        out += "{\"begin\":" + std::to_string(x.begin) + ",\"end\":" + std::to_string(x.end) + ",\"sections\":[";
        for (int i = x.begin; i <= x.end; ++i) {
            if (i > x.begin) out += ',';
            out += json::quote(p.sections[p.order[i]].id);
        }
        out += "],\"device\":" + json::quote(x.device) + ",\"layout\":" + json::quote(lstring(p, x.layout)) +
               ",\"exec_ns\":" + json::number(x.exec_ns) + "}";
    }
    return out + "]}";
}

static std::string plan_pdl(const Program& p, const Arch& a, const Profile& prof) {
    const int k = (int)p.order.size();
    std::vector<Run> R = run_nodes(p, a, prof);
    std::vector<int> order(R.size());
    for (size_t i = 0; i < R.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        if (R[x].end != R[y].end) return R[x].end < R[y].end;
        return R[x].begin < R[y].begin;
    });
    std::vector<Path> best(R.size());
    std::vector<char> has(R.size(), 0);
    for (int i : order) {
        const Run& n = R[i];
        bool got = false;
        Path cur;
        auto offer = [&](Path c) {
            if (!got || path_less(R, c, cur)) { cur = std::move(c); got = true; }
        };
        if (n.begin == 0) offer({n.exec_ns, {i}});
        for (size_t j = 0; j < R.size(); ++j) {
            const Run& m = R[j];
            if (m.end != n.begin - 1 || !has[j]) continue;
            double rc = remap_cost(p, a, m.layout, m.device, n.layout, n.device, intersect(m.fields, n.fields), nullptr);
            Path c{best[j].cost + (rc + n.exec_ns), best[j].nodes};
            c.nodes.push_back(i);
            offer(std::move(c));
        }
        if (got) { best[i] = std::move(cur); has[i] = 1; }
    }
    bool got = false;
    Path fin;
    for (size_t i = 0; i < R.size(); ++i) {
        if (R[i].end != k - 1 || !has[i]) continue;
        if (!got || path_less(R, best[i], fin)) { fin = best[i]; got = true; }
    }
    if (!got) throw PlanError(ADHA_ERR_PLANNER, "no plan covers the program");

    std::string out = "{\"schema_version\":1,\"runs\":[";
    for (size_t r = 0; r < fin.nodes.size(); ++r) {
        const Run& x = R[fin.nodes[r]];
        if (r) out += ',';
        out += "{\"sections\":[";
        for (int i = x.begin; i <= x.end; ++i) {
            if (i > x.begin) out += ',';
            out += json::quote(p.sections[p.order[i]].id);
        }
        out += "],\"device\":" + json::quote(x.device) + ",\"layout\":" + json::quote(lstring(p, x.layout)) +
               ",\"exec_ns\":" + json::number(x.exec_ns) + "}";
    }
    out += "],\"remaps\":[";
    for (size_t r = 1; r < fin.nodes.size(); ++r) {
        const Run& x = R[fin.nodes[r - 1]];
        const Run& y = R[fin.nodes[r]];
        std::vector<int> moved;
        double rc = remap_cost(p, a, x.layout, x.device, y.layout, y.device, intersect(x.fields, y.fields), &moved);
        if (r > 1) out += ',';
        out += "{\"boundary\":" + std::to_string(y.begin) +
               ",\"after\":" + json::quote(p.sections[p.order[y.begin - 1]].id) + ",\"moved\":[";
        for (size_t m = 0; m < moved.size(); ++m) {
            if (m) out += ',';
            out += json::quote(p.names[moved[m]]);
        }
        out += "],\"cost_ns\":" + json::number(rc) + "}";
    }
    out += "],\"total_ns\":" + json::number(fin.cost) + "}";
    return out;
}

static char* dup(const std::string& s) {
    char* r = (char*)std::malloc(s.size() + 1);
    if (r) std::memcpy(r, s.c_str(), s.size() + 1);
    return r;
}

}  // namespace planner
}  // namespace adha

using namespace adha;
using namespace adha::planner;

extern "C" adha_status adha_plan_ods(const char* program_json, const char* arch_json, const char* section_id,
                                     const char* device, char** layout_out) {
    clear_error();
    if (!program_json || !arch_json || !section_id || !device || !layout_out)
        return fail(ADHA_ERR_INVALID_ARG, "null argument");
    try {
        Program p = parse_program(program_json);
        Arch a = parse_arch(arch_json);
        const Section* s = nullptr;
        for (auto& x : p.sections)
            if (x.id == section_id) s = &x;
        if (!s) return fail(ADHA_ERR_PLANNER, std::string("unknown section '") + section_id + "'");
        PLayout l = ods(*s, a.dev(device), p);
        *layout_out = dup(lstring(p, l));
        if (!*layout_out) return fail(ADHA_ERR_OOM, "out of host memory");
        return ADHA_OK;
    } catch (const json::ParseError& e) {
        return fail(ADHA_ERR_PARSE, e.what());
    } catch (const PlanError& e) {
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return fail(ADHA_ERR_OOM, "out of host memory");
    }
}

extern "C" adha_status adha_plan_pdl(const char* program_json, const char* arch_json, const char* profile_json,
                                     char** plan_out) {
    clear_error();
    if (!program_json || !arch_json || !plan_out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    try {
        Program p = parse_program(program_json);
        Arch a = parse_arch(arch_json);
        Profile pr = parse_profile(profile_json);
        *plan_out = dup(plan_pdl(p, a, pr));
        if (!*plan_out) return fail(ADHA_ERR_OOM, "out of host memory");
        return ADHA_OK;
    } catch (const json::ParseError& e) {
        return fail(ADHA_ERR_PARSE, e.what());
    } catch (const PlanError& e) {
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return fail(ADHA_ERR_OOM, "out of host memory");
    }
}

extern "C" adha_status adha_plan_candidates(const char* program_json, const char* arch_json, const char* profile_json,
                                            char** runs_out) {
    clear_error();
    if (!program_json || !arch_json || !runs_out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    try {
        Program p = parse_program(program_json);
        Arch a = parse_arch(arch_json);
        Profile pr = parse_profile(profile_json);
        *runs_out = dup(candidates_json(p, a, pr));
        if (!*runs_out) return fail(ADHA_ERR_OOM, "out of host memory");
        return ADHA_OK;
    } catch (const json::ParseError& e) {
        return fail(ADHA_ERR_PARSE, e.what());
    } catch (const PlanError& e) {
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return fail(ADHA_ERR_OOM, "out of host memory");
    }
}

// vcs_host.cpp — host-side runtime of libvcs_gpu.so: errors, instance ingestion (parser,
// validation, seeded generators), the per-layer plan of the state-space builder, and the
// multi-GPU shard plan.  No device code here.
//
// Reference behaviour restated (paths relative to /root/reference/proj):
//   parse_instance / load_instance  core/src/io.cpp:51-101 (grammar io.hpp:33-40)
//   validate                        core/src/workload.cpp:35-57
//   eligibility precompute          core/src/mdp.cpp:94-116 (attr_ok, last_use_, active_)
//   random_instance                 tests/testutil.hpp:28-65 (same std::mt19937_64 and
//                                   libstdc++ uniform_int_distribution draws)
#include "vcs_internal.h"

#include <cerrno>
#include <climits>
#include <string_view>
#include <algorithm>
#include <atomic>
#include <cctype>
#include <cstring>
#include <cmath>
#include <fstream>
#include <memory>
#include <random>
#include <sstream>

namespace vcs {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t>* launches() {
    static std::atomic<uint64_t> n{0};
    return &n;
}
} // namespace

void raise(int code, const std::string& msg) { throw Error{code, msg}; }
void set_last_error(const std::string& msg) { g_last_error = msg; }
void note_launch(uint64_t n) { launches()->fetch_add(n, std::memory_order_relaxed); }
void unnote_launch(uint64_t n) { launches()->fetch_sub(n, std::memory_order_relaxed); }

void OwnedInstance::refresh_view() {
    view.n_clouds = static_cast<int32_t>(cloud_id.size());
    view.cloud_id = cloud_id.data();
    view.cloud_vm_total = cloud_vm_total.data();
    view.cloud_vm_free = cloud_vm_free.data();
    view.cloud_thr_kbps = cloud_thr.data();
    view.cloud_delay_ms = cloud_delay.data();
    view.n_tasks = static_cast<int32_t>(task_id.size());
    view.task_id = task_id.data();
    view.task_demand = task_demand.data();
    view.task_max_delay_ms = task_max_delay.data();
    view.task_min_thr_kbps = task_min_thr.data();
    view.n_bots = static_cast<int32_t>(bot_id.size());
    view.bot_id = bot_id.data();
    view.bot_task_offset = bot_off.data();
    view.beta_vc = beta_vc;
    view.beta_tc = beta_tc;
    view.gamma_vc = gamma_vc;
}

namespace {

// validate(const VccModel&) and validate(span<const BagOfTasks>), workload.cpp:35-57.
void validate(const OwnedInstance& p) {
    if (p.beta_vc < 0 || p.beta_tc < 0 || p.gamma_vc < 0)
        raise(VCS_EINVAL, "rate parameters must be non-negative");
    for (std::size_t i = 0; i < p.cloud_id.size(); ++i) {
        if (p.cloud_vm_total[i] < 0)
            raise(VCS_EINVAL, "cloud " + std::to_string(p.cloud_id[i]) + ": vm_total < 0");
        if (p.cloud_vm_free[i] < 0 || p.cloud_vm_free[i] > p.cloud_vm_total[i])
            raise(VCS_EINVAL,
                  "cloud " + std::to_string(p.cloud_id[i]) + ": vm_free outside [0, vm_total]");
    }
    for (std::size_t j = 0; j < p.task_id.size(); ++j) {
        if (p.task_demand[j] < 1)
            raise(VCS_EINVAL, "task " + std::to_string(p.task_id[j]) + ": vm_demand < 1");
        if (p.task_max_delay[j] <= 0 || p.task_min_thr[j] <= 0)
            raise(VCS_EINVAL,
                  "task " + std::to_string(p.task_id[j]) + ": requirements must be positive");
    }
}

bool skippable(const std::string& line) {
    for (char c : line) {
        if (c == '#') return true;
        if (!std::isspace(static_cast<unsigned char>(c))) return false;
    }
    return true;
}

[[noreturn]] void bad_line(int lineno, const std::string& line, const std::string& why) {
    raise(VCS_EINVAL, "line " + std::to_string(lineno) + ": " + why + " in '" + line + "'");
}

// Fast path of one well-formed directive line: whitespace-separated tokens of plain decimal
// numbers (the only forms it accepts; anything else — signs in odd places, hex, inf/nan,
// overflow, a wrong field count, a task before any bot — returns false and the line goes through
// the stream extraction below, which produces the reference's diagnostics).  For such tokens
// strtol / strtod give exactly what `>> int` / `>> double` give.
bool plain_number(const char* b, const char* e, bool integral) {
    if (b < e && (*b == '+' || *b == '-')) ++b;
    if (b == e) return false;
    bool digit = false;
    for (const char* c = b; c < e; ++c) {
        if (*c >= '0' && *c <= '9') {
            digit = true;
        } else if (integral) {
            return false;
        } else if (*c == '.' || *c == 'e' || *c == 'E' || *c == '+' || *c == '-') {
            continue;
        } else {
            return false;
        }
    }
    return digit;
}

bool fast_line(const std::string& line, OwnedInstance& p) {
    const char* tb[6];
    const char* te[6];
    int n = 0;
    const char* c = line.data();
    const char* end = c + line.size();
    while (c < end) {
        while (c < end && std::isspace(static_cast<unsigned char>(*c))) ++c;
        if (c == end) break;
        if (n == 6) return false;
        tb[n] = c;
        while (c < end && !std::isspace(static_cast<unsigned char>(*c))) ++c;
        te[n++] = c;
    }
    if (n < 2) return false;
    const std::string_view kind(tb[0], static_cast<size_t>(te[0] - tb[0]));
    auto to_int = [&](int k, int& out) {
        if (!plain_number(tb[k], te[k], true)) return false;
        char* stop = nullptr;
        errno = 0;
        const long v = std::strtol(tb[k], &stop, 10);
        if (stop != te[k] || errno == ERANGE || v < INT_MIN || v > INT_MAX) return false;
        out = static_cast<int>(v);
        return true;
    };
    auto to_double = [&](int k, double& out) {
        // an integer of <= 15 digits is exact in a double: the value strtod would return
        const char* b = tb[k];
        const bool neg = *b == '-';
        if (*b == '+' || *b == '-') ++b;
        if (te[k] - b >= 1 && te[k] - b <= 15) {
            int64_t v = 0;
            const char* q = b;
            for (; q < te[k] && *q >= '0' && *q <= '9'; ++q) v = v * 10 + (*q - '0');
            if (q == te[k]) {
                out = neg ? -static_cast<double>(v) : static_cast<double>(v);
                return true;
            }
        }
        if (!plain_number(tb[k], te[k], false)) return false;
        char* stop = nullptr;
        errno = 0;
        const double v = std::strtod(tb[k], &stop);
        if (stop != te[k] || errno == ERANGE) return false;
        out = v;
        return true;
    };
    if (kind == "task") {
        int id, demand;
        double dly, thr;
        if (n != 5 || p.bot_id.empty() || !to_int(1, id) || !to_int(2, demand) || !to_double(3, dly) ||
            !to_double(4, thr))
            return false;
        p.task_id.push_back(id);
        p.task_demand.push_back(demand);
        p.task_max_delay.push_back(dly);
        p.task_min_thr.push_back(thr);
        return true;
    }
    if (kind == "cloud") {
        int id, total;
        double thr, delay;
        if (n != 5 || !to_int(1, id) || !to_int(2, total) || !to_double(3, thr) || !to_double(4, delay))
            return false;
        p.cloud_id.push_back(id);
        p.cloud_vm_total.push_back(total);
        p.cloud_vm_free.push_back(total);
        p.cloud_thr.push_back(thr);
        p.cloud_delay.push_back(delay);
        return true;
    }
    if (kind == "bot") {
        int id;
        if (n != 2 || !to_int(1, id)) return false;
        p.bot_id.push_back(id);
        p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
        return true;
    }
    if (kind == "beta_vc" || kind == "beta_tc" || kind == "gamma_vc") {
        double v;
        if (n != 2 || !to_double(1, v)) return false;
        (kind == "beta_vc" ? p.beta_vc : kind == "beta_tc" ? p.beta_tc : p.gamma_vc) = v;
        return true;
    }
    return false;
}

void parse_into(std::istream& in, OwnedInstance& p) {
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (skippable(line)) continue;
        if (fast_line(line, p)) continue;
        std::istringstream ls(line);
        std::string kind;
        ls >> kind;
        if (kind == "beta_vc" || kind == "beta_tc" || kind == "gamma_vc") {
            double v = 0;
            if (!(ls >> v)) bad_line(lineno, line, "expected a value");
            (kind == "beta_vc" ? p.beta_vc : kind == "beta_tc" ? p.beta_tc : p.gamma_vc) = v;
        } else if (kind == "cloud") {
            int id = 0, total = 0;
            double thr = 0, delay = 0;
            if (!(ls >> id >> total >> thr >> delay))
                bad_line(lineno, line, "expected: cloud <id> <vm_total> <thr> <delay>");
            p.cloud_id.push_back(id);
            p.cloud_vm_total.push_back(total);
            p.cloud_vm_free.push_back(total); // io.cpp:71: a parsed cloud starts fully free
            p.cloud_thr.push_back(thr);
            p.cloud_delay.push_back(delay);
        } else if (kind == "bot") {
            int id = 0;
            if (!(ls >> id)) bad_line(lineno, line, "expected: bot <id>");
            p.bot_id.push_back(id);
            p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
        } else if (kind == "task") {
            if (p.bot_id.empty()) bad_line(lineno, line, "task before any bot");
            int id = 0, demand = 0;
            double dly = 0, thr = 0;
            if (!(ls >> id >> demand >> dly >> thr))
                bad_line(lineno, line, "expected: task <id> <demand> <max_delay> <min_thr>");
            p.task_id.push_back(id);
            p.task_demand.push_back(demand);
            p.task_max_delay.push_back(dly);
            p.task_min_thr.push_back(thr);
        } else {
            bad_line(lineno, line, "unknown directive '" + kind + "'");
        }
        std::string extra;
        if (ls >> extra) bad_line(lineno, line, "unexpected trailing field '" + extra + "'");
    }
    p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
    validate(p);
    p.refresh_view();
}

template <class Rng>
int draw(Rng& rng, int lo, int hi) {
    return std::uniform_int_distribution<int>(lo, hi)(rng);
}

// tests/testutil.hpp:28-65 random_instance, draw for draw.
void gen_random(std::mt19937_64& rng, int max_clouds, int max_cap, int max_tasks, int max_demand,
                OwnedInstance& p) {
    p = OwnedInstance{};
    const int n_clouds = draw(rng, 1, max_clouds);
    for (int i = 0; i < n_clouds; ++i) {
        const int cap = draw(rng, 1, max_cap);
        const int delay = draw(rng, 5, 50);
        const int thr = draw(rng, 60, 160);
        p.cloud_id.push_back(i + 1);
        p.cloud_vm_total.push_back(cap);
        p.cloud_vm_free.push_back(cap);
        p.cloud_delay.push_back(delay);
        p.cloud_thr.push_back(thr);
    }
    p.beta_vc = 1.0;
    p.beta_tc = 1.2;
    p.gamma_vc = 1.0;
    const int n_tasks = draw(rng, 1, max_tasks);
    const int n_bots = std::min(draw(rng, 1, 3), n_tasks);
    struct T { int id, demand, dly, thr; };
    std::vector<std::vector<T>> bags(static_cast<std::size_t>(n_bots));
    for (int t = 0; t < n_tasks; ++t) {
        T task;
        task.id = t + 1;
        task.demand = draw(rng, 1, max_demand);
        task.dly = draw(rng, 5, 60);
        task.thr = draw(rng, 50, 170);
        bags[static_cast<std::size_t>(t % n_bots)].push_back(task);
    }
    for (int b = 0; b < n_bots; ++b) {
        p.bot_id.push_back(b + 1);
        p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
        for (const T& task : bags[static_cast<std::size_t>(b)]) {
            p.task_id.push_back(task.id);
            p.task_demand.push_back(task.demand);
            p.task_max_delay.push_back(task.dly);
            p.task_min_thr.push_back(task.thr);
        }
    }
    p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
}

// `clouds` homogeneous clouds {vm_total cap, thr 100, delay 10} and n_tasks
// tasks {demand U[1,max_demand], max_delay 100, min_thr 50} dealt round-robin into `clouds` bags.
void gen_homog(uint64_t seed, int clouds, int cap, int n_tasks, int max_demand, OwnedInstance& p) {
    std::mt19937_64 rng(seed);
    p = OwnedInstance{};
    for (int i = 0; i < clouds; ++i) {
        p.cloud_id.push_back(i + 1);
        p.cloud_vm_total.push_back(cap);
        p.cloud_vm_free.push_back(cap);
        p.cloud_thr.push_back(100.0);
        p.cloud_delay.push_back(10.0);
    }
    const int n_bots = std::max(1, clouds);
    std::vector<std::vector<std::pair<int, int>>> bags(static_cast<std::size_t>(n_bots));
    for (int t = 0; t < n_tasks; ++t)
        bags[static_cast<std::size_t>(t % n_bots)].push_back({t + 1, draw(rng, 1, max_demand)});
    for (int b = 0; b < n_bots; ++b) {
        p.bot_id.push_back(b + 1);
        p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
        for (auto [id, demand] : bags[static_cast<std::size_t>(b)]) {
            p.task_id.push_back(id);
            p.task_demand.push_back(demand);
            p.task_max_delay.push_back(100.0);
            p.task_min_thr.push_back(50.0);
        }
    }
    p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
}

// clouds {U[50,150] VMs, thr U[60,160], delay U[5,50]} then n_bots x per_bot
// tasks {demand U[1,max_demand], max_delay U[5,60], min_thr U[50,170]}.
void gen_greedy(uint64_t seed, int clouds, int n_bots, int per_bot, int max_demand,
                OwnedInstance& p) {
    std::mt19937_64 rng(seed);
    p = OwnedInstance{};
    for (int i = 0; i < clouds; ++i) {
        const int cap = draw(rng, 50, 150);
        const int thr = draw(rng, 60, 160);
        const int delay = draw(rng, 5, 50);
        p.cloud_id.push_back(i + 1);
        p.cloud_vm_total.push_back(cap);
        p.cloud_vm_free.push_back(cap);
        p.cloud_thr.push_back(thr);
        p.cloud_delay.push_back(delay);
    }
    int id = 0;
    for (int b = 0; b < n_bots; ++b) {
        p.bot_id.push_back(b + 1);
        p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
        for (int k = 0; k < per_bot; ++k) {
            const int demand = draw(rng, 1, max_demand);
            const int dly = draw(rng, 5, 60);
            const int thr = draw(rng, 50, 170);
            p.task_id.push_back(++id);
            p.task_demand.push_back(demand);
            p.task_max_delay.push_back(dly);
            p.task_min_thr.push_back(thr);
        }
    }
    p.bot_off.push_back(static_cast<int32_t>(p.task_id.size()));
}

int bits_for(int v) {
    int b = 1;
    while (b < 31 && (1 << b) <= v) ++b;
    return b;
}

} // namespace

// Per-layer plan: attr_ok / last_use / active (mdp.cpp:94-116) plus the packed-key layout.
LayerPlan make_layer_plan(const vcs_instance* in) {
    LayerPlan pl;
    const int K = in->n_clouds, H = in->n_tasks;
    pl.horizon = H;
    pl.n_clouds = K;
    for (int i = 0; i < K; ++i)
        if (in->cloud_vm_free[i] > 0xffff)
            raise(VCS_EINVAL, "cloud free counts above 65535 are not supported");
    std::vector<std::vector<char>> attr(static_cast<std::size_t>(K));
    pl.last_use.assign(static_cast<std::size_t>(K), -1);
    for (int i = 0; i < K; ++i) {
        attr[i].assign(static_cast<std::size_t>(H), 0);
        for (int j = 0; j < H; ++j) {
            const bool ok = in->cloud_delay_ms[i] <= in->task_max_delay_ms[j] &&
                            in->cloud_thr_kbps[i] >= in->task_min_thr_kbps[j] &&
                            in->task_demand[j] <= in->cloud_vm_free[i];
            attr[i][j] = ok;
            if (ok) pl.last_use[i] = j;
        }
    }
    pl.width_of_cloud.resize(static_cast<std::size_t>(K));
    for (int i = 0; i < K; ++i)
        pl.width_of_cloud[i] = bits_for(std::max(0, in->cloud_vm_free[i]));
    pl.active.resize(static_cast<std::size_t>(H) + 1);
    pl.words.resize(static_cast<std::size_t>(H) + 1);
    pl.bit_off.resize(static_cast<std::size_t>(H) + 1);
    pl.key_bits.reserve(static_cast<std::size_t>(H) + 1);
    for (int t = 0; t <= H; ++t) {
        int na = 0;
        for (int i = 0; i < K; ++i) na += pl.last_use[i] >= t ? 1 : 0;
        pl.active[t].reserve(static_cast<std::size_t>(na)); // (one allocation per layer)
        pl.bit_off[t].reserve(static_cast<std::size_t>(na));
        for (int i = 0; i < K; ++i)
            if (pl.last_use[i] >= t) pl.active[t].push_back(i);
        if (static_cast<int>(pl.active[t].size()) > kMaxActive)
            raise(VCS_EINVAL, "more than " + std::to_string(kMaxActive) +
                                  " clouds eligible at one decision epoch are not supported");
        int cur = 0;
        for (int c : pl.active[t]) {
            const int w = pl.width_of_cloud[c];
            if ((cur % 64) + w > 64) cur = (cur / 64 + 1) * 64; // fields never straddle words
            pl.bit_off[t].push_back(static_cast<uint16_t>(cur));
            cur += w;
        }
        const int words = std::max(1, (cur + 63) / 64);
        pl.key_bits.push_back(cur);
        if (words > kMaxKeyWords)
            raise(VCS_EINVAL, "reduced state key wider than " + std::to_string(kMaxKeyWords * 64) +
                                  " bits is not supported");
        pl.words[t] = words;
    }
    pl.layers.resize(static_cast<std::size_t>(H));
    for (int t = 0; t < H; ++t) {
        LayerParam& L = pl.layers[t]; // (value-initialised by the resize: all zero)
        const auto& act = pl.active[t];
        L.n_active = static_cast<int32_t>(act.size());
        L.n_keep = static_cast<int32_t>(pl.active[t + 1].size());
        L.demand = in->task_demand[t];
        L.words = pl.words[t];
        L.next_words = pl.words[t + 1];
        const double n = static_cast<double>(L.demand);
        L.r_cloud = in->beta_vc * n;  // mdp.cpp:191 first product
        L.r_paid = -in->beta_tc * n;  // mdp.cpp:202 first product
        L.gamma = in->gamma_vc;
        // the full reward expression with nothing retired (same two rounded operations)
        L.r_cloud_kept = L.r_cloud - L.gamma * 0.0;
        L.r_paid_kept = L.r_paid - L.gamma * 0.0;
        // mixed-radix weights of layer t+1's fields (dense successor index)
        uint32_t wq[kMaxActive];
        int nwq = 0;
        uint64_t W = 1;
        for (int c : pl.active[t + 1]) {
            wq[nwq++] = static_cast<uint32_t>(W);
            W *= static_cast<uint64_t>(std::max(0, in->cloud_vm_free[c])) + 1;
            if (W > kDenseMax) break;
        }
        L.dense_size = W <= kDenseMax ? static_cast<uint32_t>(W) : 0u;
        {   // layer t's own key space, numbered like transition t-1 numbers its successors
            uint64_t Ws = 1;
            for (std::size_t p = 0; p < act.size() && Ws <= kDenseMax; ++p) {
                L.wself[p] = static_cast<uint32_t>(Ws);
                Ws *= static_cast<uint64_t>(std::max(0, in->cloud_vm_free[act[p]])) + 1;
            }
            L.self_size = Ws <= kDenseMax ? static_cast<uint32_t>(Ws) : 0u;
        }
        int kept = 0;
        for (std::size_t p = 0; p < act.size(); ++p) {
            const int c = act[p];
            L.cloud[p] = c;
            L.attr[p] = attr[c][t];
            L.width[p] = static_cast<uint8_t>(pl.width_of_cloud[c]);
            L.bit_off[p] = pl.bit_off[t][p];
            L.radix[p] = static_cast<uint32_t>(std::max(0, in->cloud_vm_free[c]) + 1);
            if (pl.last_use[c] >= t + 1) {
                L.keep_idx[p] = static_cast<int8_t>(kept);
                L.next_bit_off[p] = pl.bit_off[t + 1][kept];
                if (L.dense_size) L.wnext[p] = wq[static_cast<std::size_t>(kept)];
                ++kept;
            } else {
                L.keep_idx[p] = -1;
            }
            L.fdesc[p] = static_cast<uint32_t>(L.bit_off[p]) | (static_cast<uint32_t>(L.width[p]) << 9) |
                         (L.attr[p] ? 1u << 15 : 0u) |
                         (L.keep_idx[p] >= 0 ? (1u << 16) | (static_cast<uint32_t>(L.next_bit_off[p]) << 17) : 0u);
        }
    }
    for (int t = 1; t < H; ++t) {
        LayerParam& L = pl.layers[static_cast<std::size_t>(t)];
        bool ok = L.n_keep == L.n_active && L.n_active <= 7 && L.dense_size != 0 &&
                  L.dense_size == L.self_size;
        for (int p = 0; ok && p < L.n_active; ++p)
            ok = L.keep_idx[p] == p && L.wnext[p] == L.wself[p] && L.next_bit_off[p] == L.bit_off[p];
        L.pull = ok ? 1 : 0;
    }
    pl.init_key.assign(static_cast<std::size_t>(pl.words[0]), 0);
    for (std::size_t p = 0; p < pl.active[0].size(); ++p) {
        const int c = pl.active[0][p];
        const int off = pl.bit_off[0][p];
        pl.init_key[off / 64] |= static_cast<uint64_t>(in->cloud_vm_free[c]) << (off % 64);
    }
    return pl;
}

bool pack_key(const LayerPlan& plan, int t, const int32_t* free_vms, uint64_t* out) {
    const int words = plan.words[t];
    for (int w = 0; w < words; ++w) out[w] = 0;
    for (std::size_t p = 0; p < plan.active[t].size(); ++p) {
        const int c = plan.active[t][p];
        const int v = free_vms[c];
        const int width = plan.width_of_cloud[c];
        if (v < 0 || v > 0xffff || (width < 31 && v >= (1 << width))) return false;
        const int off = plan.bit_off[t][p];
        out[off / 64] |= static_cast<uint64_t>(v) << (off % 64);
    }
    return true;
}

} // namespace vcs

using vcs::guarded;

extern "C" {

const char* vcs_last_error(void) { return vcs::g_last_error.c_str(); }

uint64_t vcs_kernel_launches(void) { return vcs::launches()->load(); }

int vcs_instance_parse(const char* text, vcs_instance_owned** out) {
    return guarded([&] {
        auto h = std::make_unique<vcs_instance_owned>();
        std::istringstream in(text ? text : "");
        vcs::parse_into(in, h->inst);
        *out = h.release();
        return VCS_OK;
    });
}

int vcs_instance_load(const char* path, vcs_instance_owned** out) {
    return guarded([&] {
        std::ifstream in(path);
        if (!in) vcs::raise(VCS_EIO, std::string("cannot read instance file: ") + path);
        auto h = std::make_unique<vcs_instance_owned>();
        vcs::parse_into(in, h->inst);
        *out = h.release();
        return VCS_OK;
    });
}

int vcs_instance_copy(const vcs_instance* in, vcs_instance_owned** out) {
    return guarded([&] {
        auto h = std::make_unique<vcs_instance_owned>();
        auto& p = h->inst;
        const int K = in->n_clouds, T = in->n_tasks;
        p.cloud_id.assign(in->cloud_id, in->cloud_id + K);
        p.cloud_vm_total.assign(in->cloud_vm_total, in->cloud_vm_total + K);
        p.cloud_vm_free.assign(in->cloud_vm_free, in->cloud_vm_free + K);
        p.cloud_thr.assign(in->cloud_thr_kbps, in->cloud_thr_kbps + K);
        p.cloud_delay.assign(in->cloud_delay_ms, in->cloud_delay_ms + K);
        p.task_id.assign(in->task_id, in->task_id + T);
        p.task_demand.assign(in->task_demand, in->task_demand + T);
        p.task_max_delay.assign(in->task_max_delay_ms, in->task_max_delay_ms + T);
        p.task_min_thr.assign(in->task_min_thr_kbps, in->task_min_thr_kbps + T);
        if (in->n_bots > 0 && in->bot_task_offset) {
            p.bot_id.assign(in->bot_id, in->bot_id + in->n_bots);
            p.bot_off.assign(in->bot_task_offset, in->bot_task_offset + in->n_bots + 1);
        } else {
            p.bot_off.push_back(0);
            if (T > 0) {
                p.bot_id.push_back(1);
                p.bot_off.push_back(T);
            }
        }
        p.beta_vc = in->beta_vc;
        p.beta_tc = in->beta_tc;
        p.gamma_vc = in->gamma_vc;
        vcs::validate(p);
        p.refresh_view();
        *out = h.release();
        return VCS_OK;
    });
}

const vcs_instance* vcs_instance_view(const vcs_instance_owned* inst) { return &inst->inst.view; }

void vcs_instance_free(vcs_instance_owned* inst) { delete inst; }

int vcs_instance_generate(int kind, uint64_t seed, int32_t trial, int32_t a, int32_t b, int32_t c,
                          int32_t d, vcs_instance_owned** out) {
    return guarded([&] {
        auto h = std::make_unique<vcs_instance_owned>();
        if (kind == VCS_GEN_RANDOM) {
            if (a < 1 || b < 1 || c < 1 || d < 1 || trial < 0)
                vcs::raise(VCS_EINVAL, "random instance parameters must be >= 1");
            std::mt19937_64 rng(seed);
            for (int i = 0; i <= trial; ++i) vcs::gen_random(rng, a, b, c, d, h->inst);
        } else if (kind == VCS_GEN_HOMOG) {
            if (a < 0 || b < 0 || c < 0 || d < 1)
                vcs::raise(VCS_EINVAL, "homogeneous instance parameters out of range");
            vcs::gen_homog(seed, a, b, c, d, h->inst);
        } else if (kind == VCS_GEN_GREEDY) {
            if (a < 0 || b < 0 || c < 0 || d < 1)
                vcs::raise(VCS_EINVAL, "greedy instance parameters out of range");
            vcs::gen_greedy(seed, a, b, c, d, h->inst);
        } else {
            vcs::raise(VCS_EINVAL, "unknown generator kind");
        }
        h->inst.refresh_view();
        *out = h.release();
        return VCS_OK;
    });
}

// Row-block plan of the sharded solver (the B200 counterpart of BlockPartition::even,
// parallel_vi.cpp:11-24): contiguous blocks balanced on the per-state HBM cost of a sweep,
// (24 + 12 * edges/states) bytes in layer t, optionally weighted by the number of sweeps that
// visit layer t under the converged-layer skip (H - t + 1).  Results are partition-independent
// (the reference's own contract), so only the balance changes.
int vcs_shard_plan(const uint64_t* layer_offset, const uint64_t* layer_edges, int32_t horizon,
                   int32_t world, int32_t rank, int32_t skip_weighted, uint64_t* row_begin,
                   uint64_t* row_end, uint64_t* halo_begin, uint64_t* halo_end) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) vcs::raise(VCS_EINVAL, "bad world/rank");
        const int H = horizon;
        const uint64_t S = layer_offset[H + 1];
        std::vector<double> cum(static_cast<size_t>(H) + 2, 0.0); // cost before layer t
        std::vector<double> per(static_cast<size_t>(H) + 1, 0.0); // cost per state in layer t
        for (int t = 0; t <= H; ++t) {
            const double n = static_cast<double>(layer_offset[t + 1] - layer_offset[t]);
            const double e = static_cast<double>(layer_edges[t]);
            double c = n > 0 ? 24.0 + 12.0 * e / n : 0.0;
            if (skip_weighted) c *= static_cast<double>(H - t + 1);
            per[t] = c;
            cum[t + 1] = cum[t] + c * n;
        }
        auto boundary = [&](int g) -> uint64_t {
            if (g <= 0) return 0;
            if (g >= world) return S;
            const double target = cum[H + 1] * static_cast<double>(g) / static_cast<double>(world);
            int t = 0;
            while (t < H && cum[t + 1] < target) ++t;
            const uint64_t lo = layer_offset[t], hi = layer_offset[t + 1];
            if (per[t] <= 0.0) return lo;
            const double within = (target - cum[t]) / per[t];
            uint64_t b = lo + static_cast<uint64_t>(std::llround(std::max(0.0, within)));
            return std::min(b, hi);
        };
        const uint64_t rb = boundary(rank), re = std::max(rb, boundary(rank + 1));
        *row_begin = rb;
        *row_end = re;
        uint64_t hb = re, he = re;
        if (re > rb) {
            auto layer_of = [&](uint64_t row) {
                int t = 0;
                while (t < H && layer_offset[t + 1] <= row) ++t;
                return t;
            };
            const int t_first = layer_of(rb), t_last = layer_of(re - 1);
            // successors of layer t rows live in layer t+1 (mdp.cpp:190/201)
            const uint64_t succ_begin = layer_offset[std::min(t_first + 1, H + 1)];
            const uint64_t succ_end = t_last + 1 <= H ? layer_offset[t_last + 2] : layer_offset[t_last + 1];
            hb = std::max(re, succ_begin);
            he = std::max(hb, std::min(S, succ_end));
        }
        *halo_begin = hb;
        *halo_end = he;
        return VCS_OK;
    });
}

double vcs_greedy_reward(const vcs_instance* in, int64_t placed, int64_t paid, int64_t unused) {
    // greedy.cpp:32-36, same operation order.
    return in->beta_vc * static_cast<double>(placed) - in->beta_tc * static_cast<double>(paid) -
           in->gamma_vc * static_cast<double>(unused);
}

} // extern "C"

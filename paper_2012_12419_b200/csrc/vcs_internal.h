// vcs_internal.h — shared internals of libvcs_gpu.so (host C++ and CUDA translation units).
#pragma once

#include "../../include/vcs_gpu.h"

#include <cstdint>
#include <string>
#include <vector>

namespace vcs {

// ---- errors -------------------------------------------------------------------------------
// Every C entry point catches vcs::Error and returns its code; the message is kept per thread
// for vcs_last_error().
struct Error {
    int code;
    std::string msg;
};
[[noreturn]] void raise(int code, const std::string& msg);
void set_last_error(const std::string& msg);
void note_launch(uint64_t n = 1);
void unnote_launch(uint64_t n);

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host out of memory");
        return VCS_EINVAL;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return VCS_EINVAL;
    }
}

// ---- owned instance ----------------------------------------------------------------------
struct OwnedInstance {
    std::vector<int32_t> cloud_id, cloud_vm_total, cloud_vm_free;
    std::vector<double> cloud_thr, cloud_delay;
    std::vector<int32_t> task_id, task_demand;
    std::vector<double> task_max_delay, task_min_thr;
    std::vector<int32_t> bot_id, bot_off;
    double beta_vc = 1.0, beta_tc = 1.2, gamma_vc = 1.0;
    vcs_instance view{};
    void refresh_view();
};

// ---- state-space layer plan (host side of the builder) ---------------------------------------
// Maximum clouds active in one layer's reduced key, and 64-bit words per packed key.
constexpr int kMaxActive = 64;
constexpr int kMaxKeyWords = 8;

// Everything a builder kernel needs about layer t (mdp.cpp:94-151 precompute, restated per layer).
struct LayerParam {
    int32_t n_active;            // clouds in the layer-t key (active_[t].size())
    int32_t n_keep;              // clouds surviving into t+1 (= n_active of layer t+1)
    int32_t demand;              // vm_demand of task t
    int32_t words;               // packed key words of layer t
    int32_t next_words;          // packed key words of layer t+1
    int32_t pad0;
    double r_cloud;              // beta_vc * demand      (host IEEE multiply, = reference bits)
    double r_paid;               // -beta_tc * demand
    double gamma;                // penalty_per_idle_vm
    double r_cloud_kept;         // r_cloud - gamma * 0.0: reward when nothing retires
    double r_paid_kept;          // r_paid  - gamma * 0.0
    int32_t cloud[kMaxActive];   // cloud index of key position p
    int8_t attr[kMaxActive];     // attr_ok[cloud[p]][t]
    int8_t keep_idx[kMaxActive]; // position in the next key, -1 = retired at this transition
    uint16_t bit_off[kMaxActive];      // bit offset of field p in the layer-t packed key
    uint16_t next_bit_off[kMaxActive]; // bit offset of field keep_idx[p] in the next packed key
    uint8_t width[kMaxActive];   // bit width of field p
    // Dense successor index (when the layer-(t+1) key space is small): a layer-(t+1) key is a
    // vector of free-VM counts f_q in [0, free_q], so idx = sum_q f_q * W_q with mixed-radix
    // weights W_q = prod_{q' < q} (free_q' + 1) numbers the key space 0 .. dense_size-1.
    uint32_t dense_size;         // prod (free_q + 1) over layer t+1's fields; 0 = too large
    int32_t pad1;
    uint32_t wnext[kMaxActive];  // W of field keep_idx[p] in layer t+1 (0 if p retires)
    uint32_t radix[kMaxActive];  // free_{cloud[p]} + 1
    // the same numbering of layer t's OWN key space (= the successor index of transition t-1):
    // idx = sum_p f_p * wself[p]; self_size = prod radix (0 = too large)
    uint32_t wself[kMaxActive];
    uint32_t self_size;
    int32_t pull;                // 1: transition t keeps every cloud and numbers layers t and t+1
                                 // alike (wself == wnext): the builder may pull first edges
                                 // from layer t's rank table instead of pushing them (t >= 1)
    // field p in one word (the single-CTA builder reads four per shared-memory load): bits 0-8
    // bit_off, 9-14 width, 15 attr, 16 kept, 17-25 next_bit_off; 0 past n_active (a zero-width
    // retired field: it adds nothing)
    uint32_t fdesc[kMaxActive];
};

// Dense successor indices are used up to this key-space size (a 4-byte first-edge table).
constexpr uint64_t kDenseMax = 1ull << 26;

struct LayerPlan {
    int horizon = 0;
    int n_clouds = 0;
    std::vector<int> last_use;           // per cloud, -1 = never eligible
    std::vector<std::vector<int>> active; // per layer 0..H
    std::vector<LayerParam> layers;       // per layer 0..H-1 (transition t -> t+1)
    std::vector<int> words;               // packed key words per layer 0..H
    std::vector<int> key_bits;            // used bits of the packed key per layer 0..H
    std::vector<std::vector<uint16_t>> bit_off; // per layer: bit offsets of active fields
    std::vector<int> width_of_cloud;      // bit width per cloud
    std::vector<uint64_t> init_key;       // packed layer-0 key
};
LayerPlan make_layer_plan(const vcs_instance* in);
// Pack a full state's reduced key for layer t (host), or return false when a free count does
// not fit the field (the state cannot be reachable).
bool pack_key(const LayerPlan& plan, int t, const int32_t* free_vms, uint64_t* out);

} // namespace vcs

struct vcs_instance_owned {
    vcs::OwnedInstance inst;
};

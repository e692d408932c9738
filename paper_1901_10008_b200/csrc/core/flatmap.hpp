// flatmap.hpp — allocation-light containers for the decision core's hot path.
//
//   IdMap       int64 key -> int32 value, open addressing (linear probing, backward-shift
//               deletion), power-of-two capacity; no per-insert allocation.
//   SigSet      exact set of sorted int64 id lists (withheld cluster signatures,
//               scheduler.py:435-443): 64-bit hash + arena-stored members verified on hit.
#pragma once

#include <climits>
#include <cstdint>
#include <cstring>
#include <vector>

namespace gmx {

inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Hash of a short int64 sequence: one multiply-add per element, one finalizer (the element
// chain of mix64 calls it replaces cost ~6 dependent operations per element).
inline uint64_t hash_seq(uint64_t seed, const int64_t* v, size_t n) {
    uint64_t h = seed;
    for (size_t i = 0; i < n; ++i) h = (h ^ (uint64_t)v[i]) * 0x9E3779B97F4A7C15ull + (h >> 29);
    return mix64(h ^ (uint64_t)n);
}

// IdMap keys are mostly consecutive ids (kernels, requests, dispatches): a Fibonacci
// (multiplicative) hash spreads them over the table in one multiply, and the table is kept at
// most half full so linear-probe chains stay short.
class IdMap {
   public:
    IdMap() { rehash(64); }

    int32_t find(int64_t key) const {
        size_t i = home(key);
        while (slots_[i].used) {
            if (slots_[i].key == key) return slots_[i].val;
            i = (i + 1) & mask_;
        }
        return -1;
    }

    // Insert or overwrite; returns the previous value or -1 (one probe sequence).
    int32_t put(int64_t key, int32_t val) {
        if ((size_ + 1) * 2 > mask_ + 1) rehash((mask_ + 1) * 2);
        size_t i = home(key);
        while (slots_[i].used) {
            if (slots_[i].key == key) {
                const int32_t old = slots_[i].val;
                slots_[i].val = val;
                return old;
            }
            i = (i + 1) & mask_;
        }
        slots_[i] = Slot{key, val, 1};
        ++size_;
        return -1;
    }

    bool erase(int64_t key) { return take(key) != kAbsent; }

    // Remove `key` and return its value (kAbsent if it was not present): one probe sequence.
    static constexpr int64_t kAbsent = INT64_MIN;
    int64_t take(int64_t key) {
        size_t i = home(key);
        while (slots_[i].used) {
            if (slots_[i].key == key) {
                const int32_t val = slots_[i].val;
                // backward-shift deletion keeps probe chains intact without tombstones
                size_t j = i;
                for (;;) {
                    j = (j + 1) & mask_;
                    if (!slots_[j].used) break;
                    const size_t h = home(slots_[j].key);
                    const bool movable = (i <= j) ? (h <= i || h > j) : (h <= i && h > j);
                    if (movable) {
                        slots_[i] = slots_[j];
                        i = j;
                    }
                }
                slots_[i].used = 0;
                --size_;
                return val;
            }
            i = (i + 1) & mask_;
        }
        return kAbsent;
    }

    size_t size() const { return size_; }
    void clear() {
        slots_.assign(64, Slot{0, 0, 0});
        mask_ = 63;
        shift_ = 58;
        size_ = 0;
    }

   private:
    struct Slot {           // key, value and occupancy in one 16-byte entry (one cache line probe)
        int64_t key;
        int32_t val;
        int32_t used;
    };

    size_t home(int64_t key) const { return (size_t)(((uint64_t)key * 0x9E3779B97F4A7C15ull) >> shift_); }

    void rehash(size_t cap) {
        std::vector<Slot> old = std::move(slots_);
        slots_.assign(cap, Slot{0, 0, 0});
        mask_ = cap - 1;
        shift_ = 64 - __builtin_ctzll((unsigned long long)cap);
        size_ = 0;
        for (const Slot& e : old)
            if (e.used) put(e.key, e.val);
    }

    std::vector<Slot> slots_;
    size_t mask_ = 0, size_ = 0;
    int shift_ = 58;
};

class SigSet {
   public:
    SigSet() { slots_.assign(256, -1); }

    // Inserts the (sorted) id list; returns false if it was already present.
    bool insert(const int64_t* ids, int32_t n) {
        if ((count_ + 1) * 2 > slots_.size()) grow();
        const uint64_t h = hash(ids, n);
        size_t i = h & (slots_.size() - 1);
        while (slots_[i] >= 0) {
            const int32_t e = slots_[i];
            if (hashes_[e] == h && equal(e, ids, n)) return false;
            i = (i + 1) & (slots_.size() - 1);
        }
        const int32_t e = (int32_t)hashes_.size();
        hashes_.push_back(h);
        offsets_.push_back((int64_t)arena_.size());
        arena_.push_back(n);
        arena_.insert(arena_.end(), ids, ids + n);
        slots_[i] = e;
        ++count_;
        return true;
    }

    size_t size() const { return count_; }

    // Keep only the signatures for which keep(ids, n) is true (rebuilds the table).
    template <typename F>
    void retain(F keep) {
        std::vector<uint64_t> h2;
        std::vector<int64_t> off2, arena2;
        for (int32_t e = 0; e < (int32_t)hashes_.size(); ++e) {
            const int64_t* p = arena_.data() + offsets_[e];
            if (!keep(p + 1, (int32_t)p[0])) continue;
            h2.push_back(hashes_[e]);
            off2.push_back((int64_t)arena2.size());
            arena2.insert(arena2.end(), p, p + 1 + p[0]);
        }
        hashes_.swap(h2);
        offsets_.swap(off2);
        arena_.swap(arena2);
        count_ = hashes_.size();
        size_t cap = 256;
        while (cap < 2 * (count_ + 1)) cap *= 2;
        slots_.assign(cap, -1);
        for (int32_t e = 0; e < (int32_t)hashes_.size(); ++e) {
            size_t i = hashes_[e] & (slots_.size() - 1);
            while (slots_[i] >= 0) i = (i + 1) & (slots_.size() - 1);
            slots_[i] = e;
        }
    }

   private:
    static uint64_t hash(const int64_t* ids, int32_t n) {
        uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)n;
        return hash_seq(h, ids, (size_t)n);
    }
    bool equal(int32_t e, const int64_t* ids, int32_t n) const {
        const int64_t* p = arena_.data() + offsets_[e];
        return p[0] == n && std::memcmp(p + 1, ids, sizeof(int64_t) * (size_t)n) == 0;
    }
    void grow() {
        std::vector<int32_t> next(slots_.size() * 2, -1);
        for (int32_t e = 0; e < (int32_t)hashes_.size(); ++e) {
            size_t i = hashes_[e] & (next.size() - 1);
            while (next[i] >= 0) i = (i + 1) & (next.size() - 1);
            next[i] = e;
        }
        slots_.swap(next);
    }

    std::vector<int32_t> slots_;
    std::vector<uint64_t> hashes_;
    std::vector<int64_t> offsets_;
    std::vector<int64_t> arena_;
    size_t count_ = 0;
};

}  // namespace gmx

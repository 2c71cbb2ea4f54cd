// B200 drop-in: compression parameters (reference params.hpp:18-35).
// Field meaning, defaults and validation rules are the reference's; the
// checks themselves run in the C-ABI (plzgpu_validate).
#pragma once

#include <cstddef>
#include <cstdint>

namespace plz {

struct Params {
    int symbol_width = 2;                          // S in {1,2,4}
    int window = 128;                              // W in [4,255]
    int chunk_size = 2048;                         // C symbols, pow2 in [1024,16384], > W
    int interval = 1;                              // I in {1,2,4,8,16}, divides C
    std::size_t block_bytes = std::size_t{256} << 20;  // container size, multiple of C*S
    int min_match = 2;                             // derived by validate(): 2/S + 1
};

// Throws validation_error naming the offending field; returns the canonical
// Params with min_match derived.
Params validate(Params raw);

// Levels 1..4 -> windows 32/64/128/255; anything else throws validation_error.
int level_to_window(int level);

inline Params default_params() { return Params{}; }

}  // namespace plz

// Forwarder: the reference header name (include/oocnmf/synth.hpp) resolves to the B200 host core.
#pragma once
#include "oocnmf_b200/oocnmf.hpp"

"""CPU checker (TEST INFRASTRUCTURE ONLY): C restatement of the reference hot path plus the
compiled reference under oracle/_ref. Never imported by the product package."""
